"""Multi-GPU host logic for C = A.B.

C's tile row I depends only on A's tile row I and all of B, so the path
shards with exactly one exchange step:

  * partition: A by contiguous tile-row panels, boundaries from a prefix sum
    of per-row work (intermediate products, nnz(B(k,:)) summed over A's row
    entries) so skewed matrices (R-MAT) still balance; every rank computes
    the same boundaries deterministically;
  * exchange: one broadcast of B from rank 0 (NCCL over NVLink on the B200
    box, gloo in the CPU tests);
  * output: rank panels are disjoint row ranges already in global order; an
    all-gather of per-rank nnz gives each rank its global CSR offset, so the
    concatenation is byte-identical to the single-GPU result for any N.

Each rank then runs the single-GPU C-ABI path on (A panel, B).
"""
from __future__ import annotations

import numpy as np

from .tilemul import Csr


def row_work(A: Csr, B: Csr) -> np.ndarray:
    """Intermediate products of each row of A.B (C-bar per row)."""
    rownnz_b = np.diff(np.asarray(B.row_ptr)).astype(np.int64)
    contrib = rownnz_b[np.asarray(A.col)]
    cs = np.concatenate([[0], np.cumsum(contrib)])
    rp = np.asarray(A.row_ptr)
    return cs[rp[1:]] - cs[rp[:-1]]


def panel_bounds(A: Csr, B: Csr, world: int, tile: int = 16) -> list[tuple[int, int]]:
    """Tile-row aligned [r0, r1) row ranges, one per rank, of ~equal work."""
    work = row_work(A, B)
    n_tr = (A.rows + tile - 1) // tile
    per_tile_row = np.add.reduceat(work, np.arange(0, A.rows, tile)) if A.rows else np.zeros(0, np.int64)
    cum = np.concatenate([[0], np.cumsum(per_tile_row)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        # first tile row whose prefix reaches r/world of the work
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(n_tr)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n_tr))
    return [(min(int(cuts[i]) * tile, A.rows), min(int(cuts[i + 1]) * tile, A.rows)) for i in range(world)]


def take_rows(A: Csr, r0: int, r1: int) -> Csr:
    rp = np.asarray(A.row_ptr)
    lo, hi = int(rp[r0]), int(rp[r1])
    return Csr(r1 - r0, A.cols, (rp[r0:r1 + 1] - lo).astype(np.int64), np.asarray(A.col)[lo:hi],
               np.asarray(A.val)[lo:hi])


def broadcast_csr(M: Csr | None, src: int, device, dist) -> Csr:
    """Broadcast a CSR from rank `src` (torch tensors on `device`)."""
    import torch
    rank = dist.get_rank()
    meta = torch.zeros(4, dtype=torch.int64, device=device)
    if rank == src:
        meta[:] = torch.tensor([M.rows, M.cols, M.nnz, {np.dtype(np.float16): 0, np.dtype(np.float32): 1,
                                                        np.dtype(np.float64): 2}[np.asarray(M.val).dtype]])
    dist.broadcast(meta, src=src)
    rows, cols, nnz, dt = (int(x) for x in meta.tolist())
    vdt = {0: torch.float16, 1: torch.float32, 2: torch.float64}[dt]
    # one collective: row_ptr | col | val in a flat byte buffer
    esz = torch.empty(0, dtype=vdt).element_size()
    sizes = [8 * (rows + 1), 4 * nnz, esz * nnz]
    flat = torch.empty(sum(sizes), dtype=torch.uint8, device=device)
    o = [0, sizes[0], sizes[0] + sizes[1], sum(sizes)]
    rp = flat[o[0]:o[1]].view(torch.int64)
    col = flat[o[1]:o[2]].view(torch.int32)
    val = flat[o[2]:o[3]].view(vdt)
    if rank == src:
        rp.copy_(torch.from_numpy(np.ascontiguousarray(M.row_ptr, np.int64)))
        col.copy_(torch.from_numpy(np.ascontiguousarray(M.col, np.int32)))
        val.copy_(torch.from_numpy(np.ascontiguousarray(M.val)))
    dist.broadcast(flat, src=src)
    return Csr(rows, cols, rp, col, val)


def global_offsets(local_nnz: int, device, dist) -> tuple[int, int]:
    """(offset of this rank's entries in the global CSR, global nnz)."""
    import torch
    t = torch.tensor([local_nnz], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    counts = [int(x.item()) for x in out]
    r = dist.get_rank()
    return int(sum(counts[:r])), int(sum(counts))


def assemble(panels: list[Csr], cols: int) -> Csr:
    """Concatenate row panels (in rank order) into one CSR."""
    rps, colsl, vals, base = [np.zeros(1, np.int64)], [], [], 0
    for P in panels:
        rp = np.asarray(P.row_ptr)
        rps.append(rp[1:] + base)
        base += int(rp[-1])
        colsl.append(np.asarray(P.col))
        vals.append(np.asarray(P.val))
    rows = sum(P.rows for P in panels)
    return Csr(rows, cols, np.concatenate(rps), np.concatenate(colsl) if colsl else np.zeros(0, np.int32),
               np.concatenate(vals) if vals else np.zeros(0, np.float32))
