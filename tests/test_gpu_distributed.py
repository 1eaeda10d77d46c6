"""GPU, world_size 2 over gloo (both ranks on cuda:0 -- one B200 here): the
multi-GPU step of bench.py with the real CUDA library per rank.  Rank 0
broadcasts B, each rank multiplies its work-balanced A panel on the GPU
(converting only the B tile rows its panel refers to), the offsets come from
an all-gather, and the concatenated panels equal the single-call product
bit for bit.  General-row configs also run the B-summary
exchange: each rank summarises its row panel of B and the panels are
all-gathered (distributed.gather_b_summary, tsg_spgemm_bsum)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2009_14600_b200 import distributed as D
from paper_2009_14600_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_no, name, q, use_bsum=False):
    import torch
    import torch.distributed as dist
    from paper_2009_14600_b200.tilemul import Context, Csr
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mats = W.make_small(name) if name != "fem27" else W.make(name)
        A, B = mats[0], mats[1] if len(mats) > 1 else mats[0]
        Bb = D.broadcast_csr(B if rank == 0 else None, 0, "cpu", dist)
        Bd = Csr(Bb.rows, Bb.cols, Bb.row_ptr.cuda(), Bb.col.cuda(), Bb.val.cuda())
        Bh = Csr(Bb.rows, Bb.cols, Bb.row_ptr.numpy(), Bb.col.numpy(), Bb.val.numpy())
        r0, r1 = D.panel_bounds(A, Bh, world)[rank]
        ctx = Context(device=0)
        Ap = D.take_rows(A, r0, r1).to_device("cuda")
        if use_bsum:  # this rank summarises its panel of B; the panels are all-gathered
            b0, b1 = D.b_panel_bounds(Bh, world)[rank]
            part = ctx.b_summary(D.take_rows(Bh, b0, b1).to_device("cuda"))
            full = D.gather_b_summary(part, dist, "cuda")
            Cp = ctx.spgemm_bsum(Ap, Bd, full).C
            part.free()
        else:
            Cp = ctx.spgemm(Ap, Bd).C
        off, total = D.global_offsets(Cp.nnz, "cpu", dist)
        q.put((rank, off, total, Cp.row_ptr, Cp.col, Cp.val, r1 - r0))
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,use_bsum", [("fem27", False), ("rect", False), ("amg", False),
                                           ("rect", True), ("rmat", True)])
def test_two_rank_gpu_panels_equal_single_call(ctx, name, use_bsum):
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port_no = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, 2, port_no, name, q, use_bsum)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(2)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    mats = W.make_small(name) if name != "fem27" else W.make(name)
    A, B = mats[0], mats[1] if len(mats) > 1 else mats[0]
    full = ctx.spgemm(A, B).C
    from paper_2009_14600_b200.tilemul import Csr
    assert res[0][1] == 0 and res[1][1] == len(res[0][4]) and res[0][2] == full.nnz
    C = D.assemble([Csr(r[6], B.cols, r[3], r[4], r[5]) for r in res], B.cols)
    assert np.array_equal(C.row_ptr, np.asarray(full.row_ptr)) and np.array_equal(C.col, np.asarray(full.col))
    assert np.array_equal(np.asarray(C.val).view(np.uint32), np.asarray(full.val).view(np.uint32))
