"""Multi-GPU readiness on one GPU: the multi-device
context with N panel workers all on GPU 0 (tsg_create_multi with a repeated
ordinal) runs each rank's work-balanced tile-row panel of A one after
another and times each on its own stream (tsg_last_panel_ms).  The max over
panels is what an N-GPU run's compute takes (the NVLink copy of B, ~0.1-0.2
ms for R-MAT's 101 MB CSR, is not in it: the panels share GPU 0's copy).
Device-resident inputs and outputs, median of a few calls after warm-up.
Usage: python scripts/emulate_ranks.py [config ...]"""
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
    cfgs = sys.argv[1:] or ["rmat", "fem27"]
    print("| config | N | panel ms (each rank) | max | N=1 / max | balance max/mean |")
    print("|---|---|---|---|---|---|")
    for cfg in cfgs:
        mats = [dev(M) for M in W.make(cfg)]
        base = None
        for N in (1, 2, 4, 8):
            ctx = Context(devices=[0] * N)
            runs = []
            for i in range(5):
                if len(mats) == 3:
                    ctx.spgemm_chain(mats, out="device")
                else:
                    ctx.spgemm(mats[0], mats[1] if len(mats) > 1 else mats[0], out="device")
                if i >= 2:
                    runs.append(ctx.panel_ms())
            ctx.close()
            per = [statistics.median(r[p] for r in runs) for p in range(N)]
            mx = max(per)
            base = mx if N == 1 else base
            print(f"| {cfg} | {N} | {' / '.join(f'{x:.2f}' for x in per)} | {mx:.3f} | {base / mx:.2f} | "
                  f"{mx / (sum(per) / N):.2f} |", flush=True)


if __name__ == "__main__":
    main()
