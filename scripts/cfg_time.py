"""Device time per phase of one spGEMM call (device-resident inputs as
bench.py builds them), median of a few calls after warm-up.
Usage: python scripts/cfg_time.py [config ...] [--mode ordered] [--reps 5]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_14600_b200 import workloads as W  # noqa: E402
from paper_2009_14600_b200.tilemul import Context  # noqa: E402


def dev(M):
    D = M.to_device("cuda")
    h = D.val.to(torch.float16)
    return type(D)(D.rows, D.cols, D.row_ptr, D.col, h) if torch.equal(h.to(D.val.dtype), D.val) else D


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["poisson", "fem27", "amg", "rect", "rmat"])
    ap.add_argument("--mode", default="tensor")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    ctx = Context(device=0)
    for cfg in a.configs:
        mats = [dev(M) for M in W.make(cfg)]
        keys = ("convert", "task_list", "sort", "multiply", "compaction", "total")
        rows = []
        for i in range(a.reps + 2):
            if len(mats) == 3:
                r = ctx.spgemm_chain(mats, out="device", mode=a.mode, phase_timing=True)
            else:
                r = ctx.spgemm(mats[0], mats[1] if len(mats) > 1 else mats[0], out="device", mode=a.mode,
                               phase_timing=True)
            if i >= 2:
                rows.append(r.stats)
        med = {k: statistics.median(x[k] for x in rows) * 1e3 for k in keys}
        print(f"{cfg:8s} " + " ".join(f"{k}={v:.3f}" for k, v in med.items()) +
              f" nnz={rows[0]['nnz_c']} launches={rows[0]['kernel_launches']}", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
