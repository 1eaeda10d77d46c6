"""Phase times of R-MAT A.A with the same operand pointer, with a copy of A
as the left operand, and for the first (hub) 1/8 row panel -- where the
multi-device panels spend their time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_14600_b200 import distributed as D  # noqa: E402
from paper_2009_14600_b200 import workloads as W  # noqa: E402
from paper_2009_14600_b200.tilemul import Context, Csr  # noqa: E402


def dev(M):
    D_ = M.to_device("cuda")
    return Csr(D_.rows, D_.cols, D_.row_ptr, D_.col, D_.val.to(torch.float16))


ctx = Context(device=0)
A = W.make(sys.argv[1] if len(sys.argv) > 1 else "rmat")[0]
Ad = dev(A)
A2 = Csr(Ad.rows, Ad.cols, Ad.row_ptr.clone(), Ad.col.clone(), Ad.val.clone())
r0, r1 = D.panel_bounds(A, A, 8)[0]
P0 = dev(D.take_rows(A, r0, r1))
keys = ("convert", "task_list", "sort", "multiply", "compaction", "total")
for name, X in (("same", Ad), ("copy", A2), ("panel0/8", P0)):
    for i in range(3):
        r = ctx.spgemm(X, Ad, out="device", phase_timing=True)
    st = r.stats
    print(f"{name:9s} " + " ".join(f"{k}={st[k]*1e3:.3f}" for k in keys) +
          f" numeric_kernel={ctx.last_phase_ms('numeric_kernel'):.3f} path={st['path']} nnz={st['nnz_c']}"
          f" launches={st['kernel_launches']} staged={st['staged_slots']}", flush=True)

# the multi-device context with one and with eight panel workers on GPU 0
import time  # noqa: E402
for n in (1, 8):
    m = Context(devices=[0] * n)
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = m.spgemm(Ad, Ad, out="device", phase_timing=True)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    st = r.stats
    print(f"multi{n}   " + " ".join(f"{k}={st[k]*1e3:.3f}" for k in keys) + f" wall={wall:.1f}ms panel_ms=" +
          " ".join(f"{x:.2f}" for x in m.panel_ms()), flush=True)
    m.close()
