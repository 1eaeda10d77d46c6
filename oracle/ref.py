"""ctypes binding of oracle/_ref/libref_tilemul.so -- TEST INFRASTRUCTURE ONLY.

The unmodified reference (tilemul) compiled in place from /root/reference by
oracle/Makefile, behind oracle/ref_harness.cpp.  Only tests/, the smoke
check in __graft_entry__ and bench.py's CPU baseline / `--impl reference`
arm may import this; the product path never does.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "_ref" / "libref_tilemul.so"
_lib = None


def available() -> bool:
    return LIB.exists()


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise RuntimeError(f"{LIB} not built (make -C oracle ref)")
        lib = C.CDLL(str(LIB))
        P, I64 = C.c_void_p, C.c_int64
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_spgemm.argtypes = [I64, I64, P, P, P, I64, I64, P, P, P, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(P)]
        lib.ref_chain.argtypes = [C.c_int, P, P, P, P, P, C.c_int, C.c_int, C.POINTER(P)]
        lib.ref_oracle.argtypes = [C.c_int, I64, I64, P, P, P, I64, I64, P, P, P, C.POINTER(P)]
        lib.ref_tile.argtypes = [I64, I64, P, P, P, C.c_int, C.POINTER(P)]
        lib.ref_random_coo.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_int,
                                       C.POINTER(P)]
        lib.ref_corpus.argtypes = [C.c_int, C.c_int, C.POINTER(P)]
        lib.ref_round_to_half.argtypes = [C.c_double, C.POINTER(C.c_int)]
        lib.ref_round_to_half.restype = C.c_double
        lib.ref_smape.argtypes = [I64, I64, P, P, P, P, P, P]
        lib.ref_smape.restype = C.c_double
        lib.ref_result_dims.argtypes = [P, P]
        lib.ref_result_csr.argtypes = [P, P, P, P]
        lib.ref_result_tiles.argtypes = [P, P, P, P, P]
        lib.ref_result_stats.argtypes = [P, P, P, P]
        lib.ref_result_free.argtypes = [P]
        _lib = lib
    return _lib


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


@dataclass
class RefResult:
    rows: int
    cols: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray          # float64 carrier of fp32 values
    tile_row: np.ndarray     # 8x8 output tiles (reference TiledMatrix)
    tile_col: np.ndarray
    bitmap: np.ndarray
    elem_index: np.ndarray
    times: dict              # taskList, sort, counting, multiply, compaction, total (s)
    raw_pairs: int
    filtered_pairs: int
    segments: int
    counted: int
    realized: int
    threads: int
    fnv: int


def _csr_args(M):
    rp = np.ascontiguousarray(M.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(M.col, dtype=np.int32)
    val = np.ascontiguousarray(M.val, dtype=np.float64)
    return (rp, col, val), (M.rows, M.cols, rp.ctypes.data, col.ctypes.data, val.ctypes.data)


def _collect(lib, h) -> RefResult:
    dims = np.zeros(4, dtype=np.int64)
    lib.ref_result_dims(h, dims.ctypes.data)
    rows, cols, nnz, nt = (int(x) for x in dims)
    rp = np.zeros(rows + 1, dtype=np.int64)
    col = np.zeros(nnz, dtype=np.int32)
    val = np.zeros(nnz, dtype=np.float64)
    lib.ref_result_csr(h, rp.ctypes.data, col.ctypes.data, val.ctypes.data)
    tr, tc = np.zeros(nt, np.uint32), np.zeros(nt, np.uint32)
    bm, ei = np.zeros(nt, np.uint64), np.zeros(nt, np.uint64)
    lib.ref_result_tiles(h, tr.ctypes.data, tc.ctypes.data, bm.ctypes.data, ei.ctypes.data)
    t6 = np.zeros(6, np.float64)
    u6 = np.zeros(6, np.uint64)
    fnv = np.zeros(1, np.uint64)
    lib.ref_result_stats(h, t6.ctypes.data, u6.ctypes.data, fnv.ctypes.data)
    lib.ref_result_free(h)
    names = ("task_list", "sort", "counting", "multiply", "compaction", "total")
    return RefResult(rows, cols, rp, col, val, tr, tc, bm, ei, dict(zip(names, t6.tolist())),
                     int(u6[0]), int(u6[1]), int(u6[2]), int(u6[3]), int(u6[4]), int(u6[5]), int(fnv[0]))


def _check(lib, rc):
    if rc != 0:
        raise RefError(rc, lib.ref_last_error().decode())


def spgemm(A, B=None, *, threads: int = 0, pairing: bool = True) -> RefResult:
    """spgemm_square(A) when B is None, else the A.B pass composition."""
    lib = load()
    ka, a = _csr_args(A)
    kb, b = _csr_args(B if B is not None else A)
    h = C.c_void_p()
    _check(lib, lib.ref_spgemm(*a, *b, int(B is None), threads, int(pairing), C.byref(h)))
    return _collect(lib, h)


def chain(mats, *, threads: int = 0, pairing: bool = True) -> RefResult:
    lib = load()
    keep, args = zip(*[_csr_args(M) for M in mats])
    n = len(mats)
    ms = np.array([a[0] for a in args], np.int64)
    ns = np.array([a[1] for a in args], np.int64)
    rps = np.array([a[2] for a in args], np.uint64)
    cols = np.array([a[3] for a in args], np.uint64)
    vals = np.array([a[4] for a in args], np.uint64)
    h = C.c_void_p()
    _check(lib, lib.ref_chain(n, ms.ctypes.data, ns.ctypes.data, rps.ctypes.data, cols.ctypes.data,
                              vals.ctypes.data, threads, int(pairing), C.byref(h)))
    return _collect(lib, h)


def oracle(A, B=None, *, mode: str = "mixed") -> RefResult:
    """dense_spgemm_mixed_ordered (mode 'mixed') or dense_spgemm_fp64."""
    lib = load()
    ka, a = _csr_args(A)
    kb, b = _csr_args(B if B is not None else A)
    h = C.c_void_p()
    _check(lib, lib.ref_oracle(0 if mode == "mixed" else 1, *a, *b, C.byref(h)))
    return _collect(lib, h)


def tile8(M, kind: str = "fp16") -> RefResult:
    """from_element_coo(M, Fp16Stored|Fp32Stored): the reference 8x8 tiling."""
    lib = load()
    k, a = _csr_args(M)
    h = C.c_void_p()
    _check(lib, lib.ref_tile(*a, 0 if kind == "fp16" else 1, C.byref(h)))
    return _collect(lib, h)


VALUE_MODES = {"signed_halves": 0, "positive_halves": 1, "positive_reals": 2, "wild_halves": 3,
               "pattern": 4}


def random_coo(seed: int, rows: int, cols: int, density: float, mode: str = "signed_halves"):
    """make_random_coo(std::mt19937_64(seed), ...) of proj/tests/support/corpus.hpp:71-91."""
    from paper_2009_14600_b200.tilemul import Csr
    lib = load()
    h = C.c_void_p()
    _check(lib, lib.ref_random_coo(seed, rows, cols, density, VALUE_MODES[mode], C.byref(h)))
    r = _collect(lib, h)
    return Csr(r.rows, r.cols, r.row_ptr, r.col, r.val)


def corpus(which: str, index: int):
    """Matrix `index` of the acceptance corpus ('main', acceptance.cpp:45-58)
    or the WildHalves odd-dims corpus ('wild', test_kernels.cpp:332-348)."""
    from paper_2009_14600_b200.tilemul import Csr
    lib = load()
    h = C.c_void_p()
    _check(lib, lib.ref_corpus(0 if which == "main" else 1, index, C.byref(h)))
    r = _collect(lib, h)
    return Csr(r.rows, r.cols, r.row_ptr, r.col, r.val)


def round_to_half(x: float) -> float:
    lib = load()
    st = C.c_int(0)
    v = lib.ref_round_to_half(float(x), C.byref(st))
    if st.value:
        raise RefError(st.value, "round_to_half")
    return v


def smape(X, Y) -> float:
    lib = load()
    kx, x = _csr_args(X)
    ky, y = _csr_args(Y)
    return float(lib.ref_smape(x[0], x[1], x[2], x[3], x[4], y[2], y[3], y[4]))
