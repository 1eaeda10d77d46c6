"""A/B of the general-row paths on the GPU: the per-chunk shared-memory
SEaC (TSG_GENERAL=1, default) against the previous global task-list path
(TSG_GENERAL=0).  Outputs must be byte-identical, statistics equal; prints
device times.  Usage: python scripts/esc_ab.py [config ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_14600_b200 import workloads as W  # noqa: E402
from paper_2009_14600_b200.tilemul import Context  # noqa: E402


def run(ctx, mats, mode, general):
    os.environ["TSG_GENERAL"] = str(general)
    if len(mats) == 3:
        r = ctx.spgemm_chain(mats, mode=mode, phase_timing=True)
    else:
        A = mats[0]
        B = mats[1] if len(mats) > 1 else A
        r = ctx.spgemm(A, B, mode=mode, phase_timing=True)
    return r


def main():
    names = sys.argv[1:] or ["small", "rect", "amg", "rmat"]
    ctx = Context(device=0)
    for name in names:
        mats = [W.rmat(scale=12, edge_factor=16)] if name == "small" else W.make(name)
        for mode in ("tensor", "ordered"):
            rs = {}
            for gen in (1, 0):
                run(ctx, mats, mode, gen)  # warm
                t0 = time.perf_counter()
                r = run(ctx, mats, mode, gen)
                rs[gen] = (r, time.perf_counter() - t0)
            (a, ta), (b, tb) = rs[1], rs[0]
            same = (np.array_equal(a.C.row_ptr, b.C.row_ptr) and np.array_equal(a.C.col, b.C.col)
                    and np.array_equal(a.C.val.view(np.uint32), b.C.val.view(np.uint32)))
            keys = ("tiles_a", "raw_pairs", "filtered_pairs", "segments", "counted_elements", "nnz_c")
            sd = {k: (a.stats[k], b.stats[k]) for k in keys if a.stats[k] != b.stats[k]}
            print(f"{name:6s} {mode:8s} identical={same} stat_diffs={sd} "
                  f"esc_total={a.stats['total']*1e3:.3f}ms old_total={b.stats['total']*1e3:.3f}ms "
                  f"esc_mult={a.stats['multiply']*1e3:.3f} old_mult={b.stats['multiply']*1e3:.3f} "
                  f"nnz={a.stats['nnz_c']} wall {ta:.2f}/{tb:.2f}s", flush=True)
            if not same:
                for i, (x, y) in enumerate(((a.C.row_ptr, b.C.row_ptr), (a.C.col, b.C.col))):
                    if not np.array_equal(x, y):
                        j = int(np.nonzero(x != y)[0][0]) if x.shape == y.shape else -1
                        print("   first diff in", ["row_ptr", "col"][i], "at", j, x.shape, y.shape)
                        break
    ctx.close()


if __name__ == "__main__":
    main()
