"""A small parity corpus for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family runs at least once -- light and general
rows, both numeric modes, host and device output (the pipelined paths),
chains with fused emission, malformed input, the multi-device context --
and every result is checked against the reference restatement.
Usage: compute-sanitizer --tool <tool> python scripts/sanitize_corpus.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import port  # noqa: E402
from paper_2009_14600_b200 import tilemul as T  # noqa: E402
from paper_2009_14600_b200 import workloads as W  # noqa: E402


def same(a, b):
    return (np.array_equal(np.asarray(a.row_ptr), np.asarray(b.row_ptr)) and
            np.array_equal(np.asarray(a.col), np.asarray(b.col)) and
            np.array_equal(np.asarray(a.val, np.float32).view(np.uint32),
                           np.asarray(b.val, np.float32).view(np.uint32)))


def main():
    ctx = T.Context(device=0)
    n = 0
    cases = [("poisson", W.poisson2d(48)), ("fem27", W.fem27(12)), ("rmat", W.rmat(scale=11, edge_factor=8)),
             ("wide", W.random_uniform(2000, 2000, 60000, 5)), ("rowmajor", W.random_uniform(1500, 1500, 9000, 6))]
    for name, A in cases:
        want = port.spgemm_mixed(A, A)
        for mode in ("ordered", "tensor"):
            for out in ("host", "device"):
                got = ctx.spgemm(A, A, mode=mode, out=out).C
                got = got.to_numpy() if out == "device" else got
                ok = same(got, want) if mode == "ordered" or name != "wide" else \
                    np.array_equal(np.asarray(got.col), want.col)
                assert ok, (name, mode, out)
                n += 1
    R, Am, P = W.make_small("amg")
    want = port.spgemm_mixed(port.spgemm_mixed(R, Am), P)
    assert same(ctx.spgemm_chain([R, Am, P], mode="ordered").C, want)
    n += 1
    bad = W.fem27(8)
    rp = np.asarray(bad.row_ptr).copy()
    rp[-1] += 50
    try:
        ctx.spgemm(T.Csr(bad.rows, bad.cols, rp, bad.col, bad.val).to_device(), bad.to_device(), out="device")
        raise AssertionError("malformed row_ptr accepted")
    except T.InvariantError:
        n += 1
    # 8x8 re-tiling both ways (tsg_tiles8.cu)
    M = W.rmat(scale=10, edge_factor=8)
    M = T.Csr(M.rows, M.cols, M.row_ptr, M.col, np.asarray(M.val, np.float32))
    t8 = ctx.csr_to_tiles8(M)
    back = ctx.tiles8_to_csr(M.rows, M.cols, t8)
    assert np.array_equal(np.asarray(back.col), np.asarray(M.col))
    n += 1
    # B summaries of row panels, gathered, and the product through them (tsg_bsum)
    from paper_2009_14600_b200 import distributed as D
    from paper_2009_14600_b200.tilemul import BSummary
    Rm = W.rmat(scale=11, edge_factor=8)
    full = BSummary.concat([ctx.b_summary(D.take_rows(Rm, r0, r1)) for r0, r1 in D.b_panel_bounds(Rm, 3)])
    assert same(ctx.spgemm_bsum(Rm, Rm, full).C, ctx.spgemm(Rm, Rm).C)
    n += 1
    multi = T.Context(devices=[0, 0, 0])
    A = W.rmat(scale=11, edge_factor=8)
    assert same(multi.spgemm(A, A).C, ctx.spgemm(A, A).C)
    n += 1
    multi.close()
    ctx.close()
    print(f"sanitize corpus ok: {n} checked calls")


if __name__ == "__main__":
    main()
