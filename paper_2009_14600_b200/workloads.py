"""Synthetic workloads of BASELINE.json, deterministic.

All matrices are CSR with int64 row_ptr, int32 sorted columns, no
duplicates and binary16-representable float32 values.  Randomness is a
counter-based splitmix64 stream, u = (x >> 11) * 2^-53, so every host (this
container, the GPU box, each rank) regenerates identical matrices.

  1 poisson2d(256)      C = A.A, 5-point stencil, integer values
  2 fem27(64)           C = A.A, 27-point stencil, integer values (headline)
  3 rmat(20, 16)        C = A.A, R-MAT (0.45, 0.15, 0.15, 0.25), multiplicities
  4 rect()              C = A.B, 1M x 500k . 500k x 1M, 5M uniform each, U[0.5,2)
  5 amg(128)            C = (R.A).P, 7-point Laplacian 128^3, trilinear P, R = P^T
"""
from __future__ import annotations

import numpy as np

from .tilemul import Csr

_GAMMA = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """x_i = splitmix64 output number offset+i of a generator seeded `seed`."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, n: int, offset: int = 0) -> np.ndarray:
    return (splitmix64(seed, n, offset) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _from_rows_cols(n_rows: int, n_cols: int, rows: np.ndarray, cols: np.ndarray, vals: np.ndarray) -> Csr:
    """CSR from entries already sorted by (row, col), no duplicates."""
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    rp[1:] = np.cumsum(np.bincount(rows, minlength=n_rows))
    return Csr(n_rows, n_cols, rp, cols.astype(np.int32), vals.astype(np.float32))


def _stencil(dims: tuple, offsets: list, diag: float, off: float) -> Csr:
    """Grid stencil; offsets as (dz, dy, dx), no wrap.  Column order follows
    the flattened offset, so offsets are sorted by it first."""
    nz, ny, nx = dims
    n = nz * ny * nx
    offsets = sorted(offsets, key=lambda o: (o[0] * ny + o[1]) * nx + o[2])
    idx = np.arange(n, dtype=np.int64)
    z, y, x = idx // (ny * nx), (idx // nx) % ny, idx % nx
    cols = np.empty((n, len(offsets)), dtype=np.int64)
    ok = np.empty((n, len(offsets)), dtype=bool)
    vals = np.empty((n, len(offsets)), dtype=np.float32)
    for j, (dz, dy, dx) in enumerate(offsets):
        zz, yy, xx = z + dz, y + dy, x + dx
        ok[:, j] = (zz >= 0) & (zz < nz) & (yy >= 0) & (yy < ny) & (xx >= 0) & (xx < nx)
        cols[:, j] = (zz * ny + yy) * nx + xx
        vals[:, j] = diag if (dz, dy, dx) == (0, 0, 0) else off
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum(ok.sum(axis=1))
    return Csr(n, n, rp, cols[ok].astype(np.int32), vals[ok])


def poisson2d(n: int = 256) -> Csr:
    offs = [(0, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    return _stencil((1, n, n), offs, 4.0, -1.0)


def fem27(n: int = 64) -> Csr:
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
    return _stencil((n, n, n), offs, 26.0, -1.0)


def laplace7(n: int = 128) -> Csr:
    offs = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    return _stencil((n, n, n), offs, 6.0, -1.0)


def rmat(scale: int = 20, edge_factor: int = 16, abcd=(0.45, 0.15, 0.15, 0.25), seed: int = 3) -> Csr:
    """R-MAT, MSB-first quadrant bits, duplicates summed (value = multiplicity),
    self-loops kept, no permutation."""
    n = 1 << scale
    m = edge_factor * n
    a, b, c, _ = abcd
    row = np.zeros(m, dtype=np.int64)
    col = np.zeros(m, dtype=np.int64)
    for level in range(scale):
        u = uniform(seed, m, offset=level * m)
        bit = np.int64(1) << np.int64(scale - 1 - level)
        rbit = u >= a + b                      # quadrants (1,0), (1,1)
        cbit = ((u >= a) & (u < a + b)) | (u >= a + b + c)  # (0,1), (1,1)
        row |= np.where(rbit, bit, 0)
        col |= np.where(cbit, bit, 0)
    key = row * n + col
    uk, cnt = np.unique(key, return_counts=True)
    return _from_rows_cols(n, n, uk // n, uk % n, cnt.astype(np.float32))


def _round_half(x: np.ndarray) -> np.ndarray:
    return x.astype(np.float16).astype(np.float32)  # numpy casts with RNE


def random_uniform(rows: int, cols: int, nnz: int, seed: int) -> Csr:
    """Exactly `nnz` distinct uniform positions (duplicates redrawn, like
    make_random_coo, proj/tests/support/corpus.hpp:82-88); values
    PositiveHalves U[0.5, 2) rounded to binary16 (corpus.hpp:57-60)."""
    total = rows * cols
    keys = np.zeros(0, dtype=np.int64)
    drawn = 0
    while keys.size < nnz:
        need = nnz - keys.size
        x = splitmix64(seed, need, offset=drawn)
        drawn += need
        k = (x % np.uint64(total)).astype(np.int64)
        keys = np.unique(np.concatenate([keys, k]))
    vals = _round_half(0.5 + 1.5 * uniform(seed + 1, nnz))
    return _from_rows_cols(rows, cols, keys // cols, keys % cols, vals)


def rect(m: int = 1_000_000, k: int = 500_000, nnz: int = 5_000_000, seed: int = 11):
    return random_uniform(m, k, nnz, seed), random_uniform(k, m, nnz, seed + 100)


def _prolong1d(nf: int) -> tuple:
    """1D linear prolongation nf -> nf/2: weight 1 at even fine points, 1/2,1/2
    at odd points (one 1/2 at the upper boundary).  Returns (rows, cols, vals)."""
    nc = nf // 2
    r, c, v = [], [], []
    for i in range(nf):
        if i % 2 == 0:
            r.append(i), c.append(i // 2), v.append(1.0)
        else:
            for j in ((i - 1) // 2, (i + 1) // 2):
                if j < nc:
                    r.append(i), c.append(j), v.append(0.5)
    return np.array(r), np.array(c), np.array(v)


def prolongation(n: int = 128) -> Csr:
    """Trilinear P = p (x) p (x) p, fine n^3 -> coarse (n/2)^3."""
    r1, c1, v1 = _prolong1d(n)
    nc = n // 2
    # per fine 1D index: list of (coarse, weight), at most 2
    per = [[] for _ in range(n)]
    for r, c, v in zip(r1, c1, v1):
        per[r].append((c, v))
    w = max(len(p) for p in per)
    C1 = np.full((n, w), -1, dtype=np.int64)
    V1 = np.zeros((n, w), dtype=np.float64)
    for i, p in enumerate(per):
        for j, (c, v) in enumerate(p):
            C1[i, j], V1[i, j] = c, v
    # tensor product, fine index (z*n + y)*n + x, coarse (Z*nc + Y)*nc + X
    Cz = C1[:, None, None, :, None, None]
    Cy = C1[None, :, None, None, :, None]
    Cx = C1[None, None, :, None, None, :]
    cols = (Cz * nc + Cy) * nc + Cx
    ok = (Cz >= 0) & (Cy >= 0) & (Cx >= 0)
    vals = V1[:, None, None, :, None, None] * V1[None, :, None, None, :, None] * V1[None, None, :, None, None, :]
    nf = n ** 3
    cols = np.broadcast_to(cols, (n, n, n, w, w, w)).reshape(nf, w ** 3)
    ok = np.broadcast_to(ok, (n, n, n, w, w, w)).reshape(nf, w ** 3)
    vals = np.broadcast_to(vals, (n, n, n, w, w, w)).reshape(nf, w ** 3)
    # (Z,Y,X) lexicographic over the (w,w,w) block is column-sorted already
    rp = np.zeros(nf + 1, dtype=np.int64)
    rp[1:] = np.cumsum(ok.sum(axis=1))
    return Csr(nf, nc ** 3, rp, cols[ok].astype(np.int32), vals[ok].astype(np.float32))


def transpose(M: Csr) -> Csr:
    rows = np.repeat(np.arange(M.rows, dtype=np.int64), np.diff(M.row_ptr))
    order = np.lexsort((rows, M.col))
    rp = np.zeros(M.cols + 1, dtype=np.int64)
    rp[1:] = np.cumsum(np.bincount(M.col, minlength=M.cols))
    return Csr(M.cols, M.rows, rp, rows[order].astype(np.int32), M.val[order])


def amg(n: int = 128):
    """(R, A, P) of the Galerkin triple product R.A.P."""
    A = laplace7(n)
    P = prolongation(n)
    return transpose(P), A, P


def sample_tile_rows(A: Csr, stride: int) -> Csr:
    """Every `stride`-th 16-row tile row of A (a strided row sample that keeps
    the skew of the full matrix; bench.py's bounded CPU-reference sample)."""
    if stride <= 1:
        return A
    rp = np.asarray(A.row_ptr, dtype=np.int64)
    tr = np.arange(0, (A.rows + 15) // 16, stride, dtype=np.int64)
    rows = (tr[:, None] * 16 + np.arange(16, dtype=np.int64)[None, :]).ravel()
    rows = rows[rows < A.rows]
    lens = rp[rows + 1] - rp[rows]
    new_rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    # entry p of sampled row i comes from rp[rows[i]] + (p - new_rp[i])
    idx = np.repeat(rp[rows] - new_rp[:-1], lens) + np.arange(int(new_rp[-1]), dtype=np.int64)
    return Csr(len(rows), A.cols, new_rp, np.asarray(A.col)[idx], np.asarray(A.val)[idx])


def cbar(A: Csr, B: Csr) -> int:
    """sum_k nnzA(:,k) * nnzB(k,:) (analytics.cpp:51-65 generalised)."""
    colc = np.bincount(np.asarray(A.col), minlength=A.cols).astype(np.int64)
    rowc = np.diff(np.asarray(B.row_ptr)).astype(np.int64)
    return int(np.dot(colc, rowc))


CONFIGS = {
    "poisson": "C = A.A, 2D 5-point Poisson 256x256",
    "fem27": "C = A.A, 3D 27-point FEM-like stencil 64^3",
    "rmat": "C = A.A, R-MAT 2^20 rows, edge factor 16, (0.45,0.15,0.15,0.25)",
    "rect": "C = A.B, 1M x 500k . 500k x 1M, density 1e-5",
    "amg": "C = (R.A).P, 7-point Laplacian 128^3, trilinear prolongation",
}


def make_small(name: str):
    """Test-size members of each config family (same generators)."""
    if name == "poisson":
        return [poisson2d(48)]
    if name == "fem27":
        return [fem27(12)]
    if name == "rmat":
        return [rmat(scale=11, edge_factor=8)]
    if name == "rect":
        return list(rect(m=4000, k=2000, nnz=16000))
    if name == "amg":
        return list(amg(16))
    raise KeyError(name)


def make(name: str):
    """Operand list for a config: [A] for squares, [A, B], or [R, A, P]."""
    if name == "poisson":
        return [poisson2d(256)]
    if name == "fem27":
        return [fem27(64)]
    if name == "rmat":
        return [rmat()]
    if name == "rect":
        return list(rect())
    if name == "amg":
        return list(amg(128))
    raise KeyError(name)
