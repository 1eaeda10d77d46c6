"""GPU, full BASELINE sizes: each of the five configs against the C
restatement of dense_spgemm_mixed_ordered (oracle/tsg_oracle.c, pinned to
the reference by tests/test_oracle.py) and its T=16 symbolic counters.
Configs 1, 2, 3, 5 have integer / dyadic values, so TENSOR mode must be
bit-exact; config 4 (positive, ~1 product per output) pattern-exact with
values within tolerance.  Size-independent properties are checked too:
row sums (C.1 = A.(B.1)) and determinism across calls."""
import numpy as np
import pytest

from oracle import port
from paper_2009_14600_b200 import workloads as W
from tests.helpers import csr_bits_equal, csr_pattern_equal, first_diff

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not port.available(), reason="C restatement not built")]


def rowsum_check(Cm, A, B, rtol):
    ones = np.ones(B.cols)
    def spmv(M, x):
        rows = np.repeat(np.arange(M.rows), np.diff(np.asarray(M.row_ptr)))
        return np.bincount(rows, weights=np.asarray(M.val, np.float64) * x[np.asarray(M.col)], minlength=M.rows)
    want = spmv(A, spmv(B, ones))
    got = spmv(Cm, ones)
    assert np.allclose(got, want, rtol=rtol, atol=rtol)


@pytest.mark.parametrize("name", ["poisson", "fem27", "amg", "rect", "rmat"])
def test_config_full_size(ctx, name):
    mats = W.make(name)
    if len(mats) == 3:
        R, A, P = mats
        got = ctx.spgemm_chain(mats)
        want = port.spgemm_mixed(port.spgemm_mixed(R, A), P)
        assert csr_bits_equal(got.C, want), first_diff(got.C, want)
        return
    A = mats[0]
    B = mats[1] if len(mats) > 1 else A
    res = ctx.spgemm(A, B)
    res2 = ctx.spgemm(A, B)
    assert np.array_equal(res.C.col, res2.C.col) and np.array_equal(res.C.val.view(np.uint32), res2.C.val.view(np.uint32))
    want = port.spgemm_mixed(A, B)
    if name == "rect":
        assert csr_pattern_equal(res.C, want), first_diff(res.C, want)
        assert np.allclose(res.C.val, want.val, rtol=2 ** -21, atol=0)
    else:
        assert csr_bits_equal(res.C, want), first_diff(res.C, want)
    if name != "rmat":  # R-MAT (6.8e9 raw tile pairs): test_gpu_r02.py::test_rmat_full_size_t16_counters
        st16 = port.tile_stats(A, B, 16)
        for k in ("tiles_a", "raw_pairs", "filtered_pairs", "segments", "counted_elements"):
            assert res.stats[k] == st16[k], k
    assert res.stats["counted_elements"] == res.stats["nnz_c"] == want.nnz  # no cancellation
    if name != "rmat":
        rowsum_check(res.C, A, B, 1e-5)
