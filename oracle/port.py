"""ctypes binding of oracle/_ref/libtsg_oracle.so (the plain-C restatement,
oracle/tsg_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline may use it;
the product path never does.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "_ref" / "libtsg_oracle.so"
_lib = None


def available() -> bool:
    return LIB.exists()


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise RuntimeError(f"{LIB} not built (make -C oracle)")
        lib = C.CDLL(str(LIB))
        P, I64 = C.c_void_p, C.c_int64
        lib.tsgo_round_to_half.argtypes = [C.c_double, C.POINTER(C.c_int)]
        lib.tsgo_round_to_half.restype = C.c_double
        lib.tsgo_spgemm_mixed.argtypes = [I64, I64, P, P, P, I64, P, P, P, C.POINTER(P),
                                          C.POINTER(P), C.POINTER(P), C.POINTER(I64)]
        lib.tsgo_tile_stats.argtypes = [C.c_int, I64, I64, P, P, P, I64, P, P, P, P]
        lib.tsgo_fnv_tiled8.argtypes = [I64, I64, P, P, P]
        lib.tsgo_fnv_tiled8.restype = C.c_uint64
        lib.tsgo_cbar.argtypes = [I64, I64, P, P, P]
        lib.tsgo_cbar.restype = C.c_uint64
        lib.tsgo_free.argtypes = [P]
        _lib = lib
    return _lib


class PortError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"status {status}")
        self.status = status


def _arrs(M):
    rp = np.ascontiguousarray(M.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(M.col, dtype=np.int32)
    val = np.ascontiguousarray(M.val, dtype=np.float64)
    return rp, col, val


def round_to_half(x: float) -> float:
    st = C.c_int(0)
    v = load().tsgo_round_to_half(float(x), C.byref(st))
    if st.value:
        raise PortError(st.value)
    return v


def spgemm_mixed(A, B):
    """dense_spgemm_mixed_ordered restated: returns a Csr with float32 values."""
    from paper_2009_14600_b200.tilemul import Csr
    lib = load()
    a, b = _arrs(A), _arrs(B)
    rp, col, val, nnz = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_int64()
    st = lib.tsgo_spgemm_mixed(A.rows, A.cols, a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data,
                               B.cols, b[0].ctypes.data, b[1].ctypes.data, b[2].ctypes.data,
                               C.byref(rp), C.byref(col), C.byref(val), C.byref(nnz))
    if st:
        raise PortError(st)
    n = nnz.value

    def take(ptr, count, dt):
        out = np.frombuffer((C.c_char * (count * np.dtype(dt).itemsize)).from_address(ptr.value),
                            dtype=dt).copy() if count else np.zeros(0, dt)
        lib.tsgo_free(ptr)
        return out
    return Csr(A.rows, B.cols, take(rp, A.rows + 1, np.int64), take(col, n, np.int32), take(val, n, np.float32))


def tile_stats(A, B, T: int = 16) -> dict:
    lib = load()
    a, b = _arrs(A), _arrs(B)
    out = np.zeros(6, np.uint64)
    st = lib.tsgo_tile_stats(T, A.rows, A.cols, a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data,
                             B.cols, b[0].ctypes.data, b[1].ctypes.data, b[2].ctypes.data,
                             out.ctypes.data)
    if st:
        raise PortError(st)
    keys = ("tiles_a", "tiles_b", "raw_pairs", "filtered_pairs", "segments", "counted_elements")
    return {k: int(v) for k, v in zip(keys, out)}


def fnv_tiled8(Cm) -> int:
    rp = np.ascontiguousarray(Cm.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(Cm.col, dtype=np.int32)
    val = np.ascontiguousarray(Cm.val, dtype=np.float32)
    return int(load().tsgo_fnv_tiled8(Cm.rows, Cm.cols, rp.ctypes.data, col.ctypes.data, val.ctypes.data))


def cbar(A, B) -> int:
    a = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ac = np.ascontiguousarray(A.col, dtype=np.int32)
    b = np.ascontiguousarray(B.row_ptr, dtype=np.int64)
    return int(load().tsgo_cbar(A.rows, A.cols, a.ctypes.data, ac.ctypes.data, b.ctypes.data))
