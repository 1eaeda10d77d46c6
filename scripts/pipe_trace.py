"""Timeline of one host-output FEM27 call (TSG_PIPE_TRACE=1 prints the
pipelined output's milestones from the library): pinned host inputs, as in
bench.py's e2e step."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_14600_b200 import workloads as W  # noqa: E402
from paper_2009_14600_b200 import _lib as L  # noqa: E402
from paper_2009_14600_b200.tilemul import Context, Csr, _view  # noqa: E402

ctx = Context(device=0)
A = W.fem27(64)
pin = []


def pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    pin.append(t)
    return t.numpy()


h = A.val.astype(np.float16)
Ah = Csr(A.rows, A.cols, pinned(A.row_ptr), pinned(A.col), pinned(h.view(np.int16)).view(np.float16))
keep = []
av = _view(Ah, keep)
o = ctx._opts("tensor", False, False, False)
for i in range(5):
    co = L.tsg_csr_out()
    co.mem = L.TSG_MEM_HOST
    t0 = time.perf_counter()
    rc = ctx.spgemm_raw(av, av, o, co)
    t1 = time.perf_counter()
    print(f"call {i}: {1e3 * (t1 - t0):.3f} ms rc={rc}", file=sys.stderr)
    ctx.free(co)
