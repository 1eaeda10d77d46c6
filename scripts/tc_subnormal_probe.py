"""Does mma.m16n8k16 f16 honour binary16 subnormal inputs?  C = x * y for
x a subnormal (2^-24 .. 2^-15) and y = 1, 2^10; TENSOR vs ORDERED."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2009_14600_b200.tilemul import Context, Csr  # noqa: E402


def one(v):
    return Csr(16, 16, np.array([0, 1] + [1] * 15, np.int64), np.array([0], np.int32), np.array([v]))


ctx = Context()
out = []
for e in range(-24, -12):
    for y in (1.0, 1024.0):
        x = 2.0 ** e
        A, B = one(x), one(y)
        t = ctx.spgemm(A, B, mode="tensor").C
        o = ctx.spgemm(A, B, mode="ordered").C
        out.append({"x": x, "y": y, "tensor": float(t.val[0]) if t.nnz else 0.0,
                    "ordered": float(o.val[0]) if o.nnz else 0.0})
print(json.dumps(out, indent=1))
