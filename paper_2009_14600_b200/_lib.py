"""ctypes binding of the C ABI (include/tsparse_b200.h).

The CUDA library is the product path: there is no CPU fallback.  Importing
this module fails loudly when ``libtsparse_b200.so`` has not been built.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libtsparse_b200.so"

TSG_OK, TSG_ERR_OTHER, TSG_ERR_INVARIANT, TSG_ERR_OVERFLOW, TSG_ERR_DIMENSION, TSG_ERR_PRECISION = range(6)
TSG_F16, TSG_F32, TSG_F64 = 0, 1, 2
TSG_MEM_HOST, TSG_MEM_DEVICE = 0, 1
TSG_MODE_TENSOR, TSG_MODE_ORDERED = 0, 1


class tsg_csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p),
                ("dtype", C.c_int32), ("mem", C.c_int32)]


class tsg_csr_out(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p),
                ("mem", C.c_int32), ("_pad", C.c_int32), ("_owner", C.c_void_p)]


class tsg_tiles_out(C.Structure):
    _fields_ = [("ntiles", C.c_int64), ("nnz", C.c_int64),
                ("tile_row", C.c_void_p), ("tile_col", C.c_void_p), ("row_masks", C.c_void_p),
                ("elem_index", C.c_void_p), ("val", C.c_void_p)]


class tsg_tiles8(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("ntiles", C.c_int64), ("nnz", C.c_int64),
                ("tile_row", C.c_void_p), ("tile_col", C.c_void_p), ("bitmap", C.c_void_p),
                ("elem_index", C.c_void_p), ("val", C.c_void_p), ("mem", C.c_int32), ("_pad", C.c_int32)]


class tsg_tiles8_out(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("ntiles", C.c_int64), ("nnz", C.c_int64),
                ("tile_row", C.c_void_p), ("tile_col", C.c_void_p), ("bitmap", C.c_void_p),
                ("elem_index", C.c_void_p), ("val", C.c_void_p)]


class tsg_bsum(C.Structure):
    _fields_ = [("rows", C.c_int64), ("tile_rows", C.c_int64), ("tiles", C.c_int64), ("nnz", C.c_int64),
                ("njt", C.c_void_p), ("tile_count", C.c_void_p), ("rinfo", C.c_void_p), ("ro", C.c_void_p),
                ("etile", C.c_void_p), ("h16", C.c_void_p), ("_owner", C.c_void_p)]


class tsg_options(C.Structure):
    _fields_ = [("mode", C.c_int32), ("drop_nonfinite", C.c_int32),
                ("phase_timing", C.c_int32), ("want_tiles", C.c_int32)]


STAT_TIMES = ("convert", "task_list", "sort", "counting", "multiply", "compaction", "total")
STAT_COUNTS = ("tiles_a", "tiles_b", "raw_pairs", "filtered_pairs", "segments", "counted_elements",
               "nnz_c", "cbar", "kernel_launches", "h2d_bytes", "d2h_bytes",
               "staged_slots", "mem_input_tiles", "mem_input_elements", "mem_task_list", "mem_counting",
               "mem_pre_compaction", "mem_output", "mem_peak")
STAT_INTS = ("path", "devices")
TSG_PATH_PANEL, TSG_PATH_GENERAL, TSG_PATH_PANEL_EMIT = 0, 1, 2
# the numeric kernel of each path (tsg_run_stats.path)
PATH_KERNEL = {TSG_PATH_PANEL: "panel_numeric_kernel", TSG_PATH_GENERAL: "esc_kernel",
               TSG_PATH_PANEL_EMIT: "panel_numeric_kernel"}


class tsg_run_stats(C.Structure):
    _fields_ = ([(n, C.c_double) for n in STAT_TIMES] + [(n, C.c_uint64) for n in STAT_COUNTS] +
                [(n, C.c_int32) for n in STAT_INTS])

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n in STAT_TIMES + STAT_COUNTS + STAT_INTS}


# Every symbol include/tsparse_b200.h declares (checked by tests/test_abi.py).
EXPORTS = ("tsg_default_options", "tsg_create", "tsg_destroy", "tsg_last_error", "tsg_abi_version",
           "tsg_spgemm", "tsg_spgemm_chain", "tsg_free_csr", "tsg_free_tiles", "tsg_cbar",
           "tsg_launch_count", "tsg_last_kernel_ms", "tsg_create_multi", "tsg_last_panel_ms",
           "tsg_tiles8_to_csr", "tsg_csr_to_tiles8", "tsg_free_tiles8",
           "tsg_bsum_create", "tsg_bsum_free", "tsg_spgemm_bsum")

_lib = None


def load() -> C.CDLL:
    """Load the CUDA library or raise: the product path has no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: the B200 CUDA library is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
            "There is no CPU fallback for the spGEMM path.")
    lib = C.CDLL(str(LIB_PATH))
    P = C.c_void_p
    lib.tsg_default_options.argtypes = [C.POINTER(tsg_options)]
    lib.tsg_default_options.restype = None
    lib.tsg_create.argtypes = [C.POINTER(P), C.c_int, P]
    lib.tsg_create.restype = C.c_int
    lib.tsg_create_multi.argtypes = [C.POINTER(P), C.c_int, C.POINTER(C.c_int)]
    lib.tsg_create_multi.restype = C.c_int
    lib.tsg_last_panel_ms.argtypes = [P, C.POINTER(C.c_double), C.c_int]
    lib.tsg_last_panel_ms.restype = C.c_int
    lib.tsg_destroy.argtypes = [P]
    lib.tsg_destroy.restype = C.c_int
    lib.tsg_last_error.argtypes = [P]
    lib.tsg_last_error.restype = C.c_char_p
    lib.tsg_abi_version.argtypes = []
    lib.tsg_abi_version.restype = C.c_int
    lib.tsg_spgemm.argtypes = [P, C.POINTER(tsg_csr), C.POINTER(tsg_csr), C.POINTER(tsg_csr_out),
                               C.POINTER(tsg_options), C.POINTER(tsg_run_stats),
                               C.POINTER(tsg_tiles_out)]
    lib.tsg_spgemm.restype = C.c_int
    lib.tsg_spgemm_chain.argtypes = [P, C.c_int, C.POINTER(C.POINTER(tsg_csr)),
                                     C.POINTER(tsg_csr_out), C.POINTER(tsg_options),
                                     C.POINTER(tsg_run_stats)]
    lib.tsg_spgemm_chain.restype = C.c_int
    lib.tsg_free_csr.argtypes = [P, C.POINTER(tsg_csr_out)]
    lib.tsg_free_csr.restype = None
    lib.tsg_free_tiles.argtypes = [C.POINTER(tsg_tiles_out)]
    lib.tsg_free_tiles.restype = None
    lib.tsg_cbar.argtypes = [P, C.POINTER(tsg_csr), C.POINTER(tsg_csr), C.POINTER(C.c_uint64)]
    lib.tsg_cbar.restype = C.c_int
    lib.tsg_launch_count.argtypes = [P]
    lib.tsg_launch_count.restype = C.c_uint64
    lib.tsg_tiles8_to_csr.argtypes = [P, C.POINTER(tsg_tiles8), C.POINTER(tsg_csr_out)]
    lib.tsg_tiles8_to_csr.restype = C.c_int
    lib.tsg_csr_to_tiles8.argtypes = [P, C.POINTER(tsg_csr), C.POINTER(tsg_tiles8_out)]
    lib.tsg_csr_to_tiles8.restype = C.c_int
    lib.tsg_free_tiles8.argtypes = [C.POINTER(tsg_tiles8_out)]
    lib.tsg_free_tiles8.restype = None
    lib.tsg_bsum_create.argtypes = [P, C.POINTER(tsg_csr), C.POINTER(tsg_bsum)]
    lib.tsg_bsum_create.restype = C.c_int
    lib.tsg_bsum_free.argtypes = [P, C.POINTER(tsg_bsum)]
    lib.tsg_bsum_free.restype = None
    lib.tsg_spgemm_bsum.argtypes = [P, C.POINTER(tsg_csr), C.POINTER(tsg_csr), C.POINTER(tsg_bsum),
                                    C.POINTER(tsg_csr_out), C.POINTER(tsg_options), C.POINTER(tsg_run_stats)]
    lib.tsg_spgemm_bsum.restype = C.c_int
    lib.tsg_last_kernel_ms.argtypes = [P, C.c_char_p]
    lib.tsg_last_kernel_ms.restype = C.c_double
    _lib = lib
    return lib
