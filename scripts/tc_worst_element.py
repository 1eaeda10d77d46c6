"""Find the worst TENSOR-mode element of a golden WildHalves case and print
its products (diagnostic)."""
import sys
from fractions import Fraction

import numpy as np

sys.path.insert(0, ".")
from paper_2009_14600_b200.tilemul import Context  # noqa: E402
from tests import golden_io as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "wild_00"
d = G.load(name)
A = G.csr(d, "A")
want = G.expected(d, "oracle").C
ctx = Context()
got = ctx.spgemm(A, A, mode="tensor").C
Ah = A.val.astype(np.float16).astype(np.float64)
rows = np.repeat(np.arange(want.rows), np.diff(want.row_ptr))
worst, wi = -1.0, -1
for i in range(want.nnz):
    r, c = rows[i], want.col[i]
    prods = []
    for p in range(A.row_ptr[r], A.row_ptr[r + 1]):
        k = A.col[p]
        for q in range(A.row_ptr[k], A.row_ptr[k + 1]):
            if A.col[q] == c:
                prods.append((k, Ah[p] * Ah[q]))
    s = sum(abs(x) for _, x in prods)
    err = abs(float(got.val[i]) - want.val[i])
    ratio = err / (2 * len(prods) * 2.0 ** -23 * s) if s else 0
    if ratio > worst:
        worst, wi, wp = ratio, i, prods
r, c = rows[wi], want.col[wi]
exact = sum(Fraction(x) for _, x in wp)
print(f"{name}: worst ratio {worst:.2f} at ({r},{c}); n={len(wp)}")
print(f"  tensor {float(got.val[wi])!r}  ordered/ref {want.val[wi]!r}  exact {float(exact)!r}")
for k, x in wp:
    print(f"   k={k:4d} (tile {k//16}) product {x!r}")
