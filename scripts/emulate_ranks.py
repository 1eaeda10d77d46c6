"""Multi-GPU readiness on one GPU: every rank's call of
an N-GPU run, timed alone.  Rank p's operands are its work-balanced tile-row
panel of A (paper_2009_14600_b200/distributed.py panel_bounds, the split
bench.py and tsg_create_multi use) and the full B, device-resident; its
device time is the library's own event bracket (tsg_run_stats.total, median
of 3 after warm-up).  The max over ranks is the compute time of the N-GPU
step; the broadcast of B (R-MAT: 101 MB of CSR, ~0.1-0.2 ms over NVLink) is
not included.  
General configs (rmat, rect) also run the B-summary exchange
(distributed.gather_b_summary): rank p summarises its row panel of B
(tsg_bsum_create, its device time from the library's event bracket), the
panels are all-gathered (NOT measurable on one GPU: the time shown is the
bytes a rank receives at 600 GB/s plus 20 us -- NCCL all-gather on NVLink 5
/ NVSwitch), and the rank's product reads B through the gathered summary
(tsg_spgemm_bsum, library event bracket) instead of converting all of B.
Usage: python scripts/emulate_ranks.py [config ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_14600_b200 import distributed as D  # noqa: E402
from paper_2009_14600_b200 import workloads as W  # noqa: E402
from paper_2009_14600_b200.tilemul import Context, Csr  # noqa: E402


def dev(M):
    Dm = M.to_device("cuda")
    h = Dm.val.to(torch.float16)
    return Csr(Dm.rows, Dm.cols, Dm.row_ptr, Dm.col, h) if torch.equal(h.to(Dm.val.dtype), Dm.val) else Dm


def call(ctx, mats):
    if len(mats) == 3:
        return ctx.spgemm_chain(mats, out="device", phase_timing=True).stats
    return ctx.spgemm(mats[0], mats[1], out="device", phase_timing=True).stats


def main():
    cfgs = sys.argv[1:] or ["rmat", "fem27", "amg"]
    ctx = Context(device=0)
    base_ms = {}
    print("| config | N | per-rank ms (convert + rest) | max | N=1 / max | max / mean |")
    print("|---|---|---|---|---|---|")
    for cfg in cfgs:
        host = W.make(cfg)
        A, rest = host[0], host[1:] if len(host) > 1 else host[:1]
        rest_d = [dev(M) for M in rest]
        base = None
        for N in (1, 2, 4, 8):
            per, conv = [], []
            for r0, r1 in D.panel_bounds(A, rest[0], N):
                square = len(host) == 1
                # N = 1 of a square product is the plain A.A call (one operand, converted once)
                mats = ([rest_d[0]] if N == 1 and square else [dev(D.take_rows(A, r0, r1))]) + rest_d
                runs = []
                for i in range(5):
                    st = call(ctx, mats)
                    if i >= 2:
                        runs.append((st["total"] * 1e3, st["convert"] * 1e3))
                per.append(statistics.median(x[0] for x in runs))
                conv.append(statistics.median(x[1] for x in runs))
                del mats
                torch.cuda.empty_cache()
            mx = max(per)
            base = mx if N == 1 else base
            base_ms[cfg] = base
            cells = " / ".join(f"{t:.2f} ({c:.2f})" for t, c in zip(per, conv))
            print(f"| {cfg} | {N} | {cells} | {mx:.3f} | {base / mx:.2f} | {mx / (sum(per) / N):.2f} |", flush=True)
    for cfg in [c for c in cfgs if c in ("rmat", "rect")]:
        bsum_table(ctx, cfg, base_ms[cfg])
    ctx.close()


GATHER_GBS, GATHER_LAT_MS = 600.0, 0.02


def bsum_table(ctx, cfg, base):
    """Ratios against the plain one-GPU call (base, ms: A.A converts A once)."""
    from paper_2009_14600_b200.tilemul import BSummary
    host = W.make(cfg)
    A, B = host[0], host[1] if len(host) > 1 else host[0]
    B_d = dev(B)
    print(f"\n| {cfg} (B summaries) | N | per-rank ms: summary + gather (est.) + call | max | N=1 / max |")
    print("|---|---|---|---|---|")
    print(f"| {cfg} | 1 | plain call | {base:.3f} | 1.00 |")
    for N in (2, 4, 8):
        parts, t_sum = [], []
        for r0, r1 in D.b_panel_bounds(B, N):
            Bp = dev(D.take_rows(B, r0, r1))
            runs = []
            for i in range(4):
                s = ctx.b_summary(Bp)
                if i >= 1:
                    runs.append(ctx.last_phase_ms("bsum"))  # device time (library event bracket)
                if i < 3:
                    s.free()
            parts.append(s)
            t_sum.append(statistics.median(runs))
        full = BSummary.concat(parts)
        cells, tot = [], []
        for p, (r0, r1) in enumerate(D.panel_bounds(A, B, N)):
            Ap = dev(D.take_rows(A, r0, r1))
            runs = []
            for i in range(5):
                st = ctx.spgemm_bsum(Ap, B_d, full, out="device", phase_timing=True).stats
                if i >= 2:
                    runs.append(st["total"] * 1e3)
            t_call = statistics.median(runs)
            recv = full.nbytes() - parts[p].nbytes()
            t_g = recv / (GATHER_GBS * 1e6) + GATHER_LAT_MS
            t_s = max(t_sum)  # the gather waits for the slowest panel
            tot.append(t_s + t_g + t_call)
            cells.append(f"{t_s:.2f} + {t_g:.2f} + {t_call:.2f}")
        for p in parts:
            p.free()
        mx = max(tot)
        print(f"| {cfg} | {N} | {' / '.join(cells)} | {mx:.3f} | {base / mx:.2f} |", flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
