"""CPU, world_size 2 over gloo: the multi-GPU host logic (panel partition,
B broadcast, global offsets, assembly) reproduces the single-process
product byte for byte.  The per-rank compute here is the C restatement
(test stand-in for the GPU call each rank makes on the B200 box)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import port
from paper_2009_14600_b200 import distributed as D
from paper_2009_14600_b200 import workloads as W

pytestmark = pytest.mark.skipif(not port.available(), reason="C restatement not built")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_no, name, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mats = W.make_small(name)
        A, B = mats[0], mats[1] if len(mats) > 1 else mats[0]
        Bb = D.broadcast_csr(B if rank == 0 else None, 0, "cpu", dist)  # torch CPU tensors
        Bh = type(B)(Bb.rows, Bb.cols, Bb.row_ptr.numpy(), Bb.col.numpy(), Bb.val.numpy())
        bounds = D.panel_bounds(A, Bh, world)
        r0, r1 = bounds[rank]
        Cp = port.spgemm_mixed(D.take_rows(A, r0, r1), Bh)
        off, total = D.global_offsets(Cp.nnz, "cpu", dist)
        q.put((rank, bounds, off, total, Cp.row_ptr, Cp.col, Cp.val))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["fem27", "rect", "rmat"])
def test_two_rank_panels_reassemble_exactly(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mats = W.make_small(name)
    A, B = mats[0], mats[1] if len(mats) > 1 else mats[0]
    full = port.spgemm_mixed(A, B)
    bounds = res[0][1]
    assert bounds == res[1][1] and bounds[0][0] == 0 and bounds[-1][1] == A.rows
    assert all(b[0] % 16 == 0 for b in bounds)
    assert res[0][2] == 0 and res[1][2] == len(res[0][5]) and res[0][3] == full.nnz
    from paper_2009_14600_b200.tilemul import Csr
    panels = [Csr(bounds[r][1] - bounds[r][0], B.cols, res[r][4], res[r][5], res[r][6]) for r in range(2)]
    C = D.assemble(panels, B.cols)
    assert np.array_equal(C.row_ptr, full.row_ptr) and np.array_equal(C.col, full.col)
    assert np.array_equal(C.val.view(np.uint32), full.val.view(np.uint32))


def test_panel_bounds_balance_skewed_rows():
    A = W.make_small("rmat")[0]
    b = D.panel_bounds(A, A, 4)
    work = D.row_work(A, A)
    per = [int(work[r0:r1].sum()) for r0, r1 in b]
    assert b[0][0] == 0 and b[-1][1] == A.rows
    assert max(per) <= 1.5 * (sum(per) / 4) + int(work.max()) * 16


def _bsum_worker(rank, world, port_no, name, q):
    import torch
    import torch.distributed as dist
    from paper_2009_14600_b200.tilemul import BSUM_ARRAYS, BSummary
    from tests.helpers import bsum_reference
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mats = W.make_small(name)
        B = mats[1] if len(mats) > 1 else mats[0]
        bounds = D.b_panel_bounds(B, world)
        r0, r1 = bounds[rank]
        ref = bsum_reference(D.take_rows(B, r0, r1))
        arrays = {n: torch.from_numpy(np.ascontiguousarray(ref[n]).view(np.int32 if ts == "<i4" else np.int16))
                  for n, _, ts in BSUM_ARRAYS}
        full = D.gather_b_summary(BSummary(*ref["dims"], arrays), dist, "cpu")
        q.put((rank, bounds, (full.rows, full.tile_rows, full.tiles, full.nnz),
               {n: full.arrays[n].numpy().copy() for n, _, _ in BSUM_ARRAYS}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["rect", "rmat"])
def test_b_summary_all_gather_equals_whole_b(name):
    """Every rank summarises its row panel of B; the all-gathered panels are the
    summary of all of B (tsg_bsum, tests/helpers.bsum_reference)."""
    from tests.helpers import bsum_reference
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_bsum_worker, args=(r, world, port_no, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mats = W.make_small(name)
    B = mats[1] if len(mats) > 1 else mats[0]
    ref = bsum_reference(B)
    for rank, bounds, dims, arrays in res:
        assert bounds[0][0] == 0 and bounds[-1][1] == B.rows and all(b[0] % 16 == 0 for b in bounds)
        assert dims == ref["dims"]
        for n in arrays:
            want = ref[n].view(np.int32 if ref[n].dtype == np.uint32 else np.int16)
            assert np.array_equal(arrays[n], want), (rank, n)


def _bcast_worker(rank, world, port_no, q):
    import torch.distributed as dist
    from paper_2009_14600_b200.tilemul import Csr
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp = np.array([0, 2, 3, 5], np.int64)  # odd nnz with float64 values: the val section must stay aligned
        M = Csr(3, 4, rp, np.array([0, 3, 1, 0, 2], np.int32), np.array([1.5, -2.0, 3.25, 4.0, -0.5]))
        B = D.broadcast_csr(M if rank == 0 else None, 0, "cpu", dist)
        q.put((rank, B.row_ptr.numpy().tolist(), B.col.numpy().tolist(), B.val.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_broadcast_csr_float64_odd_nnz():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, rp, col, val in res:
        assert rp == [0, 2, 3, 5] and col == [0, 3, 1, 0, 2] and val == [1.5, -2.0, 3.25, 4.0, -0.5]
