"""Python mirror of the reference's hot-path API, over the C ABI.

The reference (tilemul, /root/reference/proj) exposes the spGEMM path as C++:
``spgemm_square(A)`` (proj/include/tilemul/kernels.hpp:88-89) over
``from_element_coo`` / ``to_element_coo`` (tile_format.hpp:71-75) and the
exception taxonomy of errors.hpp:9-51.  This module keeps those names and
their error behaviour, with CSR (== sorted duplicate-free COO) as the
interchange format, so the parity tests read like the reference's tests:

    C = spgemm_square(A)          # DimensionError for non-square A
    C = spgemm(A, B)              # DimensionError when A.cols != B.rows
    C = spgemm_chain([R, A, P])   # binary16 downcast between stages

Every call runs the sm_100a CUDA path (libtsparse_b200.so); there is no CPU
fallback.  C++ users get the same names from include/tilemul_gpu.hpp.
"""
from __future__ import annotations

import builtins
import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class Error(RuntimeError):
    """tilemul::Error (errors.hpp:9-11)."""


class InvariantError(Error):
    """tilemul::InvariantError: unsorted / duplicated / out-of-range input."""


class OverflowError(Error):  # noqa: A001 - mirrors tilemul::OverflowError
    """tilemul::OverflowError: value outside the binary16 finite range."""


class DimensionError(Error):
    """tilemul::DimensionError: inner dimensions differ / non-square."""


class PrecisionError(Error):
    """tilemul::PrecisionError: non-finite accumulator."""


_STATUS = {L.TSG_ERR_INVARIANT: InvariantError, L.TSG_ERR_OVERFLOW: OverflowError,
           L.TSG_ERR_DIMENSION: DimensionError, L.TSG_ERR_PRECISION: PrecisionError}


@dataclass
class Csr:
    """CSR matrix: numpy arrays (host) or torch CUDA tensors (device)."""
    rows: int
    cols: int
    row_ptr: object
    col: object
    val: object

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    @property
    def on_device(self) -> bool:
        return hasattr(self.val, "is_cuda") and bool(self.val.is_cuda)

    def to_numpy(self) -> "Csr":
        if not self.on_device:
            return self
        return Csr(self.rows, self.cols, self.row_ptr.cpu().numpy(), self.col.cpu().numpy(),
                   self.val.cpu().numpy())

    def to_device(self, device: str = "cuda") -> "Csr":
        import torch
        if self.on_device:
            return self
        return Csr(self.rows, self.cols, torch.from_numpy(np.ascontiguousarray(self.row_ptr)).to(device),
                   torch.from_numpy(np.ascontiguousarray(self.col)).to(device),
                   torch.from_numpy(np.ascontiguousarray(self.val)).to(device))

    def nbytes(self) -> int:
        return int(self.row_ptr.nbytes + self.col.nbytes + self.val.nbytes) if not self.on_device else \
            int(self.row_ptr.numel() * 8 + self.col.numel() * 4 + self.val.numel() * self.val.element_size())


@dataclass
class Tiles:
    """16x16 tiled view of C (pre-CSR, compacted): the tile-structure bridge."""
    tile_row: np.ndarray
    tile_col: np.ndarray
    row_masks: np.ndarray  # (ntiles, 16) uint16, bit c of row r = slot (r, c)
    elem_index: np.ndarray
    val: np.ndarray


@dataclass
class Result:
    C: Csr
    stats: dict = field(default_factory=dict)
    tiles: Tiles | None = None


_DT = {np.dtype(np.float16): L.TSG_F16, np.dtype(np.float32): L.TSG_F32, np.dtype(np.float64): L.TSG_F64}


def _view(M: Csr, keep: list) -> L.tsg_csr:
    v = L.tsg_csr()
    v.rows, v.cols, v.nnz = int(M.rows), int(M.cols), int(M.nnz)
    if M.on_device:
        import torch
        tdt = {torch.float16: L.TSG_F16, torch.float32: L.TSG_F32, torch.float64: L.TSG_F64}
        rp = M.row_ptr.contiguous().to(torch.int64)
        col = M.col.contiguous().to(torch.int32)
        val = M.val.contiguous()
        keep += [rp, col, val]
        # the conversions above (and whatever produced M) are queued on torch's
        # current stream; the library runs on its own stream, so they must be
        # complete before it reads the arrays
        torch.cuda.current_stream(val.device).synchronize()
        v.row_ptr, v.col, v.val = rp.data_ptr(), col.data_ptr(), val.data_ptr()
        v.dtype = tdt[val.dtype]
        v.mem = L.TSG_MEM_DEVICE
    else:
        rp = np.ascontiguousarray(M.row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(M.col, dtype=np.int32)
        val = np.ascontiguousarray(M.val)
        if val.dtype not in _DT:
            val = val.astype(np.float64)
        keep += [rp, col, val]
        v.row_ptr, v.col, v.val = rp.ctypes.data, col.ctypes.data, val.ctypes.data
        v.dtype = _DT[val.dtype]
        v.mem = L.TSG_MEM_HOST
    return v


def _np_from(ptr: int, n: int, dtype) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=dtype)
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype).copy()


class Context:
    """One tsg_ctx (device + stream + memory pool).  One per host thread.

    ``devices=[d0, d1, ...]`` makes a multi-device context (tsg_create_multi):
    every call splits A into len(devices) work-balanced tile-row panels, one
    per listed GPU (an ordinal may repeat), and concatenates the result."""

    def __init__(self, device: int = -1, stream: int | None = None, devices: list | None = None):
        self._lib = L.load()
        h = C.c_void_p()
        if devices is not None:
            arr = (C.c_int * len(devices))(*devices)
            rc = self._lib.tsg_create_multi(C.byref(h), len(devices), arr)
        else:
            rc = self._lib.tsg_create(C.byref(h), device, C.c_void_p(stream) if stream else None)
        self.n_panels = len(devices) if devices is not None else 1
        if rc != L.TSG_OK:
            raise Error(f"tsg_create failed ({rc})")
        self._h = h
        self._fin = weakref.finalize(self, self._lib.tsg_destroy, h)

    def close(self):
        self._fin()

    @property
    def handle(self):
        return self._h

    def _raise(self, rc: int):
        msg = self._lib.tsg_last_error(self._h).decode()
        raise _STATUS.get(rc, Error)(msg)

    def _opts(self, mode, phase_timing, want_tiles, drop_nonfinite) -> L.tsg_options:
        o = L.tsg_options()
        self._lib.tsg_default_options(C.byref(o))
        o.mode = {"tensor": L.TSG_MODE_TENSOR, "ordered": L.TSG_MODE_ORDERED}[mode]
        o.phase_timing = int(bool(phase_timing))
        o.want_tiles = int(bool(want_tiles))
        o.drop_nonfinite = int(bool(drop_nonfinite))
        return o

    def _collect(self, out: L.tsg_csr_out, device: bool) -> Csr:
        if device:
            import torch
            n, r = int(out.nnz), int(out.rows)
            # copy into torch-owned memory, then release the library buffers
            rp = _cuda_tensor(out.row_ptr, r + 1, torch.int64).clone()
            col = _cuda_tensor(out.col, n, torch.int32).clone() if n else torch.zeros(0, dtype=torch.int32, device="cuda")
            val = _cuda_tensor(out.val, n, torch.float32).clone() if n else torch.zeros(0, dtype=torch.float32, device="cuda")
            torch.cuda.synchronize()
            res = Csr(int(out.rows), int(out.cols), rp, col, val)
        else:
            res = Csr(int(out.rows), int(out.cols), _np_from(out.row_ptr, int(out.rows) + 1, np.int64),
                      _np_from(out.col, int(out.nnz), np.int32), _np_from(out.val, int(out.nnz), np.float32))
        self._lib.tsg_free_csr(self._h, C.byref(out))
        return res

    def spgemm(self, A: Csr, B: Csr, *, mode: str = "tensor", out: str = "host",
               want_tiles: bool = False, phase_timing: bool = False,
               drop_nonfinite: bool = False) -> Result:
        keep: list = []
        a = _view(A, keep)
        b = a if B is A else _view(B, keep)
        o = self._opts(mode, phase_timing, want_tiles, drop_nonfinite)
        co = L.tsg_csr_out()
        co.mem = L.TSG_MEM_DEVICE if out == "device" else L.TSG_MEM_HOST
        st = L.tsg_run_stats()
        to = L.tsg_tiles_out()
        rc = self._lib.tsg_spgemm(self._h, C.byref(a), C.byref(b), C.byref(co), C.byref(o),
                                  C.byref(st), C.byref(to))
        if rc != L.TSG_OK:
            self._raise(rc)
        res = Result(self._collect(co, out == "device"), st.as_dict())
        if want_tiles:
            nt, nz = int(to.ntiles), int(to.nnz)
            res.tiles = Tiles(_np_from(to.tile_row, nt, np.uint32), _np_from(to.tile_col, nt, np.uint32),
                              _np_from(to.row_masks, nt * 16, np.uint16).reshape(nt, 16),
                              _np_from(to.elem_index, nt, np.uint64), _np_from(to.val, nz, np.float32))
            self._lib.tsg_free_tiles(C.byref(to))
        return res

    def b_summary(self, B: Csr) -> "BSummary":
        """B's share of a general-row product for a row panel of B (its own
        CSR, row_ptr from 0, first row a multiple of 16 in B): tsg_bsum_create.
        The arrays are device tensors on this context's GPU."""
        keep: list = []
        b = _view(B, keep)
        s = L.tsg_bsum()
        rc = self._lib.tsg_bsum_create(self._h, C.byref(b), C.byref(s))
        if rc != L.TSG_OK:
            self._raise(rc)
        return BSummary.from_struct(s, self)

    def spgemm_bsum(self, A: Csr, B: Csr, bsum: "BSummary", *, mode: str = "tensor", out: str = "host",
                    phase_timing: bool = False, drop_nonfinite: bool = False) -> Result:
        """C = A.B with B's summary given (tsg_spgemm_bsum), e.g. gathered
        from every rank's panel (distributed.gather_b_summary)."""
        keep: list = []
        a = _view(A, keep)
        b = _view(B, keep)
        sv = bsum.struct()
        o = self._opts(mode, phase_timing, False, drop_nonfinite)
        co = L.tsg_csr_out()
        co.mem = L.TSG_MEM_DEVICE if out == "device" else L.TSG_MEM_HOST
        st = L.tsg_run_stats()
        rc = self._lib.tsg_spgemm_bsum(self._h, C.byref(a), C.byref(b), C.byref(sv), C.byref(co), C.byref(o),
                                       C.byref(st))
        if rc != L.TSG_OK:
            self._raise(rc)
        return Result(self._collect(co, out == "device"), st.as_dict())

    def spgemm_bsum_raw(self, a: L.tsg_csr, b: L.tsg_csr, bsum: "BSummary", o: L.tsg_options,
                        co: L.tsg_csr_out, st: L.tsg_run_stats | None = None) -> int:
        """tsg_spgemm_bsum without wrapping (benchmarking; caller frees `co`)."""
        sv = bsum.struct()
        return self._lib.tsg_spgemm_bsum(self._h, C.byref(a), C.byref(b), C.byref(sv), C.byref(co), C.byref(o),
                                         C.byref(st) if st is not None else None)

    def spgemm_raw(self, a: L.tsg_csr, b: L.tsg_csr, o: L.tsg_options, co: L.tsg_csr_out,
                   st: L.tsg_run_stats | None = None) -> int:
        """Zero-overhead call for benchmarking (caller frees `co`)."""
        return self._lib.tsg_spgemm(self._h, C.byref(a), C.byref(b), C.byref(co), C.byref(o),
                                    C.byref(st) if st is not None else None, None)

    def free(self, co: L.tsg_csr_out):
        self._lib.tsg_free_csr(self._h, C.byref(co))

    def spgemm_chain(self, mats: list, *, mode: str = "tensor", out: str = "host",
                     phase_timing: bool = False) -> Result:
        keep: list = []
        views = [_view(M, keep) for M in mats]
        arr = (C.POINTER(L.tsg_csr) * len(views))(*[C.pointer(v) for v in views])
        o = self._opts(mode, phase_timing, False, False)
        co = L.tsg_csr_out()
        co.mem = L.TSG_MEM_DEVICE if out == "device" else L.TSG_MEM_HOST
        st = L.tsg_run_stats()
        rc = self._lib.tsg_spgemm_chain(self._h, len(views), arr, C.byref(co), C.byref(o), C.byref(st))
        if rc != L.TSG_OK:
            self._raise(rc)
        return Result(self._collect(co, out == "device"), st.as_dict())

    def cbar(self, A: Csr, B: Csr) -> int:
        keep: list = []
        a, b = _view(A, keep), _view(B, keep)
        v = C.c_uint64()
        rc = self._lib.tsg_cbar(self._h, C.byref(a), C.byref(b), C.byref(v))
        if rc != L.TSG_OK:
            self._raise(rc)
        return int(v.value)

    def csr_to_tiles8(self, M: Csr) -> dict:
        """8x8 tiles of a CSR on the GPU (from_element_coo(Fp32Stored) of it):
        dict of numpy arrays tile_row, tile_col, bitmap, elem_index, val."""
        keep: list = []
        v = _view(Csr(M.rows, M.cols, M.row_ptr, M.col,
                      M.val.to(__import__("torch").float32) if M.on_device else np.asarray(M.val, np.float32)), keep)
        out = L.tsg_tiles8_out()
        rc = self._lib.tsg_csr_to_tiles8(self._h, C.byref(v), C.byref(out))
        if rc != L.TSG_OK:
            self._raise(rc)
        nt, nz = int(out.ntiles), int(out.nnz)
        res = {"tile_row": _np_from(out.tile_row, nt, np.uint32), "tile_col": _np_from(out.tile_col, nt, np.uint32),
               "bitmap": _np_from(out.bitmap, nt, np.uint64), "elem_index": _np_from(out.elem_index, nt, np.uint64),
               "val": _np_from(out.val, nz, np.float32)}
        self._lib.tsg_free_tiles8(C.byref(out))
        return res

    def tiles8_to_csr(self, rows: int, cols: int, t: dict, out: str = "host") -> Csr:
        """CSR of 8x8 tiles (arrays as csr_to_tiles8 returns them: numpy, or
        torch CUDA tensors of the same element sizes) on the GPU."""
        names = (("tile_row", np.uint32), ("tile_col", np.uint32), ("bitmap", np.uint64),
                 ("elem_index", np.uint64), ("val", np.float32))
        device = hasattr(t["val"], "is_cuda") and t["val"].is_cuda
        v = L.tsg_tiles8()
        if device:
            import torch
            torch.cuda.current_stream(t["val"].device).synchronize()  # the library's stream reads after torch's writes
            arr = {k: t[k].contiguous() for k, _ in names}
            for k, dt in names:
                assert arr[k].element_size() == np.dtype(dt).itemsize, k
            ptr = {k: a.data_ptr() for k, a in arr.items()}
            n_t, n_e = arr["tile_row"].numel(), arr["val"].numel()
            v.mem = L.TSG_MEM_DEVICE
        else:
            arr = {k: np.ascontiguousarray(t[k], dt) for k, dt in names}
            ptr = {k: a.ctypes.data for k, a in arr.items()}
            n_t, n_e = len(arr["tile_row"]), len(arr["val"])
            v.mem = L.TSG_MEM_HOST
        v.rows, v.cols, v.ntiles, v.nnz = rows, cols, n_t, n_e
        for k, _ in names:
            setattr(v, k, ptr[k])
        co = L.tsg_csr_out()
        co.mem = L.TSG_MEM_DEVICE if out == "device" else L.TSG_MEM_HOST
        rc = self._lib.tsg_tiles8_to_csr(self._h, C.byref(v), C.byref(co))
        if rc != L.TSG_OK:
            self._raise(rc)
        return self._collect(co, out == "device")

    def launch_count(self) -> int:
        return int(self._lib.tsg_launch_count(self._h))

    def last_phase_ms(self, phase: str) -> float:
        return float(self._lib.tsg_last_kernel_ms(self._h, phase.encode()))

    def panel_ms(self) -> list:
        """Per-panel device times (ms) of the last call of a multi-device context."""
        buf = (C.c_double * max(1, self.n_panels))()
        k = self._lib.tsg_last_panel_ms(self._h, buf, self.n_panels)
        return [float(buf[i]) for i in range(k)]


# (array, its length field, element typestr): the tsg_bsum arrays (u32 / u16 carried as i4 / i2)
BSUM_ARRAYS = (("njt", "rows", "<i4"), ("tile_count", "tile_rows", "<i4"), ("rinfo", "tile_rows", "<i4"),
               ("ro", "tiles", "<i2"), ("etile", "nnz", "<i4"), ("h16", "nnz", "<i2"))


class BSummary:
    """A B summary (tsg_bsum) as device tensors: one row panel's (library
    owned until free()) or the row-order concatenation of several panels'."""

    def __init__(self, rows: int, tile_rows: int, tiles: int, nnz: int, arrays: dict, owner=None):
        self.rows, self.tile_rows, self.tiles, self.nnz = rows, tile_rows, tiles, nnz
        self.arrays = arrays
        self._owner = owner  # (context, tsg_bsum) of a library-owned summary

    @classmethod
    def from_struct(cls, s: L.tsg_bsum, ctx: "Context") -> "BSummary":
        import torch
        dims = {"rows": s.rows, "tile_rows": s.tile_rows, "tiles": s.tiles, "nnz": s.nnz}
        arrays = {}
        for name, dim, ts in BSUM_ARRAYS:
            n = int(dims[dim])
            arrays[name] = torch.as_tensor(_CAI(getattr(s, name), n, ts), device="cuda") if n else \
                torch.zeros(0, dtype=torch.int32 if ts == "<i4" else torch.int16, device="cuda")
        return cls(int(s.rows), int(s.tile_rows), int(s.tiles), int(s.nnz), arrays, owner=(ctx, s))

    @classmethod
    def concat(cls, parts: list) -> "BSummary":
        """Panels in row order -> the summary of all their rows (every array
        is per row, per tile row, per tile or per entry, in that order)."""
        import torch
        arrays = {name: torch.cat([p.arrays[name] for p in parts]) for name, _, _ in BSUM_ARRAYS}
        return cls(sum(p.rows for p in parts), sum(p.tile_rows for p in parts), sum(p.tiles for p in parts),
                   sum(p.nnz for p in parts), arrays)

    def struct(self) -> L.tsg_bsum:
        s = L.tsg_bsum()
        s.rows, s.tile_rows, s.tiles, s.nnz = self.rows, self.tile_rows, self.tiles, self.nnz
        for name, _, _ in BSUM_ARRAYS:
            t = self.arrays[name]
            setattr(s, name, t.data_ptr() if t.numel() else None)
        return s

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.arrays.values())

    def free(self):
        if self._owner is not None:
            ctx, s = self._owner
            self.arrays = {}
            ctx._lib.tsg_bsum_free(ctx.handle, C.byref(s))
            self._owner = None


class _CAI:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _cuda_tensor(ptr, n, dtype):
    import torch
    ts = {torch.int64: "<i8", torch.int32: "<i4", torch.float32: "<f4"}[dtype]
    return torch.as_tensor(_CAI(ptr, n, ts), device="cuda")


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context()
    return _default


def spgemm(A: Csr, B: Csr, **kw) -> Csr:
    """C = A.B (the pass composition of proj/tests/test_kernels.cpp:197-202)."""
    return default_context().spgemm(A, B, **kw).C


def spgemm_square(A: Csr, **kw) -> Csr:
    """C = A.A; DimensionError for non-square input (kernels.cpp:223-226)."""
    if A.rows != A.cols:
        raise DimensionError(f"matrix squaring needs a square input, got {A.rows}x{A.cols}")
    return default_context().spgemm(A, A, **kw).C


def spgemm_chain(mats: list, **kw) -> Csr:
    """X0.X1...Xn-1 left to right with the binary16 downcast between stages."""
    return default_context().spgemm_chain(mats, **kw).C


__all__ = ["Error", "InvariantError", "OverflowError", "DimensionError", "PrecisionError", "Csr",
           "Tiles", "Result", "Context", "spgemm", "spgemm_square", "spgemm_chain", "default_context"]
_ = builtins  # builtins.OverflowError stays reachable as builtins.OverflowError
