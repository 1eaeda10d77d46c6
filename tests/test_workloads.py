"""CPU: the synthetic BASELINE workloads are well-formed CSR with the
sizes SURVEY.md 8(d) states (C-bar always computed, never hard-coded)."""
import numpy as np
import pytest

from paper_2009_14600_b200 import workloads as W


def well_formed(M):
    rp, col, val = np.asarray(M.row_ptr), np.asarray(M.col), np.asarray(M.val)
    assert rp[0] == 0 and rp[-1] == col.size == val.size and np.all(np.diff(rp) >= 0)
    assert col.size == 0 or (col.min() >= 0 and col.max() < M.cols)
    rows = np.repeat(np.arange(M.rows), np.diff(rp))
    key = rows.astype(np.int64) * M.cols + col
    assert np.all(np.diff(key) > 0)  # sorted, no duplicates
    assert np.all(val != 0) and np.all(val.astype(np.float16).astype(np.float32) == val)  # binary16 values


def test_splitmix_is_counter_based():
    a = W.splitmix64(5, 10)
    b = W.splitmix64(5, 6, offset=4)
    assert np.array_equal(a[4:], b)
    u = W.uniform(9, 100000)
    assert 0 <= u.min() and u.max() < 1 and abs(u.mean() - 0.5) < 0.01


def test_poisson_and_fem27_sizes():
    P = W.poisson2d(256)
    well_formed(P)
    assert P.nnz == 326656 and W.cbar(P, P) == 1629192
    F = W.fem27(64)
    well_formed(F)
    assert F.nnz == 6859000 and W.cbar(F, F) == 181321496


def test_amg_operators():
    R, A, P = W.amg(128)
    well_formed(A)
    well_formed(P)
    assert A.nnz == 14581760 and P.nnz == 6967871 and (R.rows, R.cols) == (262144, 2097152)
    assert W.cbar(R, A) == 48556211
    Rs, As, Ps = W.amg(8)
    dense_p = np.zeros((Ps.rows, Ps.cols))
    for i in range(Ps.rows):
        dense_p[i, Ps.col[Ps.row_ptr[i]:Ps.row_ptr[i + 1]]] = Ps.val[Ps.row_ptr[i]:Ps.row_ptr[i + 1]]
    dense_r = np.zeros((Rs.rows, Rs.cols))
    for i in range(Rs.rows):
        dense_r[i, Rs.col[Rs.row_ptr[i]:Rs.row_ptr[i + 1]]] = Rs.val[Rs.row_ptr[i]:Rs.row_ptr[i + 1]]
    assert np.array_equal(dense_r, dense_p.T)
    # a fine point with all coordinates even copies one coarse value; row sums
    # are 1 except where an odd coordinate sits on the upper boundary (1/2 each)
    assert Ps.row_ptr[1] == 1 and Ps.col[0] == 0 and Ps.val[0] == 1.0
    assert set(np.round(dense_p.sum(axis=1), 6)) <= {1.0, 0.5, 0.25, 0.125}


@pytest.mark.parametrize("name", ["poisson", "fem27", "rmat", "rect", "amg"])
def test_small_families_well_formed(name):
    for M in W.make_small(name):
        well_formed(M)


def test_rect_exact_nnz_and_rmat_multiplicities():
    A, B = W.rect(m=20000, k=10000, nnz=30000)
    assert A.nnz == B.nnz == 30000
    assert (A.rows, A.cols, B.rows, B.cols) == (20000, 10000, 10000, 20000)
    R = W.rmat(scale=12, edge_factor=16)
    well_formed(R)
    assert R.val.sum() == 16 * (1 << 12)  # duplicates summed into multiplicities
