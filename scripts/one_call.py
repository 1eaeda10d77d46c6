"""One spGEMM call on device-resident inputs of a bench config (for ncu
captures: every kernel launched here belongs to that single call)."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2009_14600_b200 import workloads as W  # noqa: E402
from paper_2009_14600_b200.tilemul import Context  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "fem27"
mode = sys.argv[2] if len(sys.argv) > 2 else "tensor"
ctx = Context(device=0)
def dev(M):
    """Device CSR as bench.py builds it: binary16 values as fp16 when exact."""
    D = M.to_device("cuda")
    h = D.val.to(torch.float16)
    return type(D)(D.rows, D.cols, D.row_ptr, D.col, h) if torch.equal(h.to(D.val.dtype), D.val) else D


host = W.make(cfg)
if os.environ.get("ONE_CALL_PANEL"):  # "N,p": rank p's panel of an N-GPU run (A rows), full B
    from paper_2009_14600_b200 import distributed as Dist
    N, p = (int(x) for x in os.environ["ONE_CALL_PANEL"].split(","))
    A = host[0]
    B = host[1] if len(host) > 1 else host[0]
    r0, r1 = Dist.panel_bounds(A, B, N)[p]
    host = [Dist.take_rows(A, r0, r1), B] + list(host[2:])
mats = [dev(M) for M in host]
bsum = None
if os.environ.get("ONE_CALL_BSUM"):  # B through its summary (assembled from N row panels), as an N-GPU rank
    from paper_2009_14600_b200 import distributed as Dist
    from paper_2009_14600_b200.tilemul import BSummary
    Bfull = W.make(cfg)[1] if len(W.make(cfg)) > 1 else W.make(cfg)[0]
    nb = int(os.environ["ONE_CALL_BSUM"])
    parts = []
    for r0, r1 in Dist.b_panel_bounds(Bfull, nb):
        parts.append(ctx.b_summary(dev(Dist.take_rows(Bfull, r0, r1))))
        print("bsum panel", r0, r1, "ms", round(ctx.last_phase_ms("bsum"), 4))
    bsum = BSummary.concat(parts)
torch.cuda.synchronize()


def call():
    if bsum is not None:
        return ctx.spgemm_bsum(mats[0], mats[1] if len(mats) > 1 else mats[0], bsum, out="device", mode=mode)
    if len(mats) == 3:
        return ctx.spgemm_chain(mats, out="device", mode=mode)
    return ctx.spgemm(mats[0], mats[1] if len(mats) > 1 else mats[0], out="device", mode=mode)


if os.environ.get("ONE_CALL_WARM") == "1":  # a first call sizes the staging arena (the speculative path runs next)
    call()
    torch.cuda.synchronize()
r = call()
torch.cuda.synchronize()
print(cfg, r.stats["nnz_c"])
