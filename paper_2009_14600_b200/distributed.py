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

General rows (R-MAT, the rectangular product) read B through its CSR plus a
B summary (tsg_bsum: per-row / per-tile-row / per-tile / per-entry arrays of
B's 16x16 tiling).  Rather than every rank converting all of B, rank p
summarises its own row panel of B (b_panel_bounds) and the panels are
all-gathered into the summary of B (gather_b_summary): the conversion work is
split N ways and the exchange is one all-gather of ~6 bytes per entry.
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


UNIT_PRODUCTS = 3584  # products per general-path work unit (tsg_kernels.cuh kEscTarget)
SEARCH_WEIGHT = 0.9   # cost of one (A entry, work unit) range search, in products


def panel_bounds(A: Csr, B: Csr, world: int, tile: int = 16) -> list[tuple[int, int]]:
    """Tile-row aligned [r0, r1) row ranges, one per rank, of ~equal work.
    A tile row's work is its intermediate products plus, for the general
    path, the range searches of its work units: every unit (~UNIT_PRODUCTS
    products) searches the B rows of all the tile row's A entries, which
    makes hub tile rows (R-MAT's first rows) cost more than their products
    (measured: rank 0 of 8 took 9% longer with products balanced alone)."""
    work = row_work(A, B)
    n_tr = (A.rows + tile - 1) // tile
    starts = np.arange(0, A.rows, tile)
    prod = np.add.reduceat(work, starts).astype(np.float64) if A.rows else np.zeros(0)
    ent = np.add.reduceat(np.diff(np.asarray(A.row_ptr)), starts).astype(np.float64) if A.rows else np.zeros(0)
    per_tile_row = prod + np.floor(SEARCH_WEIGHT * np.ceil(prod / UNIT_PRODUCTS) * ent)  # (tsg_api.cu panel_cost)
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
    sizes = [8 * (rows + 1), (4 * nnz + 7) // 8 * 8, esz * nnz]  # col padded: f64 values stay 8-byte aligned
    flat = torch.empty(sum(sizes), dtype=torch.uint8, device=device)
    o = [0, sizes[0], sizes[0] + sizes[1], sum(sizes)]
    rp = flat[o[0]:o[1]].view(torch.int64)
    col = flat[o[1]:o[1] + 4 * nnz].view(torch.int32)
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


def b_panel_bounds(B: Csr, world: int, tile: int = 16) -> list[tuple[int, int]]:
    """Tile-row aligned [r0, r1) row ranges of B, one per rank, of ~equal nnz
    (each rank summarises one, gather_b_summary)."""
    rp = np.asarray(B.row_ptr, dtype=np.int64)
    n_tr = (B.rows + tile - 1) // tile
    cum = rp[np.minimum(np.arange(n_tr + 1) * tile, B.rows)]
    cuts = [0] + [int(np.searchsorted(cum, cum[-1] * r / world, side="left")) for r in range(1, world)] + [n_tr]
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n_tr))
    return [(min(int(cuts[i]) * tile, B.rows), min(int(cuts[i + 1]) * tile, B.rows)) for i in range(world)]


def gather_b_summary(part, dist, device):
    """All-gather every rank's B-panel summary (tilemul.BSummary) and
    concatenate them in rank (= row) order: one collective on a flat byte
    buffer per rank (its six arrays back to back, padded to the largest)."""
    import torch
    from .tilemul import BSUM_ARRAYS, BSummary
    world = dist.get_world_size()
    dims = torch.tensor([part.rows, part.tile_rows, part.tiles, part.nnz], dtype=torch.int64, device=device)
    all_dims = [torch.zeros_like(dims) for _ in range(world)]
    dist.all_gather(all_dims, dims)
    all_dims = [[int(x) for x in d.tolist()] for d in all_dims]
    field = {"rows": 0, "tile_rows": 1, "tiles": 2, "nnz": 3}

    def layout(d):  # byte offsets of the arrays of a rank with dims d
        offs, o = [], 0
        for _, dim, ts in BSUM_ARRAYS:
            n = d[field[dim]] * (4 if ts == "<i4" else 2)
            offs.append((o, n))
            o += (n + 15) // 16 * 16
        return offs, o

    sizes = [layout(d)[1] for d in all_dims]
    maxb = max(max(sizes), 16)
    offs, _ = layout(all_dims[dist.get_rank()])
    flat = torch.zeros(maxb, dtype=torch.uint8, device=device)
    for (name, _, _), (o, n) in zip(BSUM_ARRAYS, offs):
        if n:
            flat[o:o + n].copy_(part.arrays[name].contiguous().view(torch.uint8))
    out = torch.empty(world * maxb, dtype=torch.uint8, device=device)
    if flat.is_cuda and dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, flat)
    else:  # gloo (CPU tests, shared-GPU runs): staged through host memory
        host = torch.empty(world * maxb, dtype=torch.uint8)
        dist.all_gather(list(host.view(world, maxb)), flat.cpu())
        out.copy_(host)
    parts = []
    for r, d in enumerate(all_dims):
        ro, _ = layout(d)
        base = r * maxb
        arrays = {}
        for (name, _, ts), (o, n) in zip(BSUM_ARRAYS, ro):
            arrays[name] = out[base + o:base + o + n].view(torch.int32 if ts == "<i4" else torch.int16)
        parts.append(BSummary(d[0], d[1], d[2], d[3], arrays))
    return BSummary.concat(parts)
