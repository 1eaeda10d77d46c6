"""Characterise the fp32 accumulation of mma.m16n8k16 f16 on this GPU through
the product path: C(0,0) = 1 + s*2^-k computed by the TENSOR mode vs exact.

Prints, for each k, the TENSOR result and the sequential-fp32 result, and
the smallest k at which the small term is lost, within one MMA (both terms
in one 16-wide k block) and across MMAs (terms in different tile pairs)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2009_14600_b200.tilemul import Context, Csr  # noqa: E402


def csr_from_dense(D):
    rows, cols = np.nonzero(D)
    rp = np.zeros(D.shape[0] + 1, np.int64)
    rp[1:] = np.cumsum(np.bincount(rows, minlength=D.shape[0]))
    return Csr(D.shape[0], D.shape[1], rp, cols.astype(np.int32), D[rows, cols].astype(np.float64))


def probe(ctx, k, sign, across):
    n = 32 if across else 16
    A = np.zeros((16, n))
    B = np.zeros((n, 16))
    A[0, 0] = 1.0
    j = 16 if across else 1  # second term in the next tile (k block) or the same one
    A[0, j] = sign * 2.0 ** -k if k <= 24 else 0.0
    B[0, 0] = 1.0
    B[j, 0] = 1.0
    if k > 24:  # build 2^-k as a product of two binary16 values
        A[0, j] = sign * 2.0 ** -12
        B[j, 0] = 2.0 ** -(k - 12)
    C = ctx.spgemm(csr_from_dense(A), csr_from_dense(B), mode="tensor").C
    Co = ctx.spgemm(csr_from_dense(A), csr_from_dense(B), mode="ordered").C
    v = float(C.val[0]) if C.nnz and C.col[0] == 0 else 0.0
    vo = float(Co.val[0]) if Co.nnz and Co.col[0] == 0 else 0.0
    return v, vo


def main():
    ctx = Context()
    out = {}
    for across in (False, True):
        for sign in (1, -1):
            rows = []
            for k in range(18, 36):
                v, vo = probe(ctx, k, sign, across)
                rows.append({"k": k, "tensor": v.hex(), "ordered": vo.hex(), "exact": (1 + sign * 2.0 ** -k).hex()})
            out[f"{'across' if across else 'within'}_{'+' if sign > 0 else '-'}"] = rows
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
