import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2009_14600_b200 import workloads as W
from paper_2009_14600_b200.tilemul import Context
ctx = Context(device=0)
A = W.fem27(64)
for i in range(4):
    t0 = time.time(); r = ctx.spgemm(A, A); print("call", i, round((time.time()-t0)*1e3, 3), "ms", file=sys.stderr)
