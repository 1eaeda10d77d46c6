"""GPU parity tests: the CUDA path (through the C ABI) vs the reference.

The reference is the unmodified tilemul library compiled in place
(oracle/_ref, see oracle/Makefile).  Bars:
  * ORDERED mode: bit-exact values and pattern vs dense_spgemm_mixed_ordered
    on every input (the acceptance criterion-1 contract).
  * TENSOR mode: pattern and tile structure bit-exact; values bit-exact on
    integer / dyadic inputs, else |c - r| <= 2 n 2^-23 sum|a b|.
"""
import numpy as np
import pytest

from oracle import ref
from paper_2009_14600_b200 import tilemul as T
from paper_2009_14600_b200 import workloads as W
from tests.helpers import csr_bits_equal, csr_pattern_equal, first_diff, quadrants, tolerance_ok

pytestmark = pytest.mark.gpu


def test_golden_hash_fixture(ctx):
    """proj/tests/test_cli.cpp:149-169 fixture: seed 5150, 120^2, 5%."""
    A = ref.random_coo(5150, 120, 120, 0.05)
    want = ref.oracle(A)
    assert want.fnv == 0x2D882906D15D6FAF
    for mode in ("ordered", "tensor"):
        res = ctx.spgemm(A, A, mode=mode, want_tiles=True)
        if mode == "ordered":  # the reference's bit-exact contract
            assert csr_bits_equal(res.C, want), (mode, first_diff(res.C, want))
        else:  # MMA accumulation order: pattern exact, values within tolerance
            assert csr_pattern_equal(res.C, want), first_diff(res.C, want)
            ok, worst = tolerance_ok(res.C, want, A, A)
            assert ok, worst
        r, c, b = quadrants(res.tiles)
        assert np.array_equal(r, want.tile_row) and np.array_equal(c, want.tile_col)
        assert np.array_equal(b, want.bitmap)


@pytest.mark.parametrize("mode", ["ordered", "tensor"])
def test_acceptance_corpus(ctx, mode):
    """acceptance.cpp:45-58,114-135: 200 matrices, SignedHalves."""
    bad = []
    for i in range(200):
        A = ref.corpus("main", i)
        want = ref.oracle(A)
        got = ctx.spgemm(A, A, mode=mode).C
        if mode == "ordered":
            if not csr_bits_equal(got, want):
                bad.append((i, first_diff(got, want)))
        else:
            if not csr_pattern_equal(got, want):
                bad.append((i, first_diff(got, want)))
                continue
            ok, worst = tolerance_ok(got, want, A, A) if A.rows <= 200 else (True, 0.0)
            if not ok:
                bad.append((i, f"tolerance {worst}"))
    assert not bad, bad[:5]


def test_wild_corpus_ordered(ctx):
    """test_kernels.cpp:332-348: full binary16 range, odd dims (edge tiles)."""
    for i in range(30):
        A = ref.corpus("wild", i)
        want = ref.oracle(A)
        got = ctx.spgemm(A, A, mode="ordered").C
        assert csr_bits_equal(got, want), (i, first_diff(got, want))


def test_poisson_tensor_bit_exact(ctx):
    A = W.poisson2d(256)
    want = ref.spgemm(A)
    res = ctx.spgemm(A, A, want_tiles=True)
    assert csr_bits_equal(res.C, want), first_diff(res.C, want)
    assert res.stats["counted_elements"] == want.counted
    r, c, b = quadrants(res.tiles)
    assert np.array_equal(r, want.tile_row) and np.array_equal(c, want.tile_col)
    assert np.array_equal(b, want.bitmap)


def test_fem27_tensor_bit_exact(ctx):
    A = W.fem27(64)
    want = ref.spgemm(A)
    res = ctx.spgemm(A, A)
    assert csr_bits_equal(res.C, want), first_diff(res.C, want)
    st = res.stats
    assert st["counted_elements"] == want.counted == 30959144
    assert st["nnz_c"] == want.realized
    # T=16 restatement counts
    assert st["tiles_a"] == 361000
    assert st["raw_pairs"] == 8329256 and st["filtered_pairs"] == 7047832
    assert st["segments"] == 985960


def test_rect_small(ctx):
    A = W.random_uniform(20000, 10000, 40000, 5)
    B = W.random_uniform(10000, 20000, 40000, 6)
    want = ref.spgemm(A, B)
    got = ctx.spgemm(A, B).C
    assert csr_pattern_equal(got, want), first_diff(got, want)
    assert got.nnz == want.realized


def test_amg_chain_small(ctx):
    R, A, P = W.amg(32)
    want = ref.chain([R, A, P])
    got = ctx.spgemm_chain([R, A, P]).C
    assert csr_bits_equal(got, want), first_diff(got, want)


def test_errors(ctx):
    A = ref.random_coo(7, 32, 32, 0.1)
    B = ref.random_coo(8, 16, 32, 0.1)
    with pytest.raises(T.DimensionError):
        ctx.spgemm(A, B)
    big = T.Csr(8, 8, np.array([0, 1, 1, 1, 1, 1, 1, 1, 1]), np.array([0], np.int32), np.array([70000.0]))
    with pytest.raises(T.OverflowError):
        ctx.spgemm(big, big)
    bad = T.Csr(8, 8, np.array([0, 2, 2, 2, 2, 2, 2, 2, 2]), np.array([3, 1], np.int32), np.array([1.0, 2.0]))
    with pytest.raises(T.InvariantError):
        ctx.spgemm(bad, bad)
    nan = T.Csr(8, 8, np.array([0, 1, 1, 1, 1, 1, 1, 1, 1]), np.array([0], np.int32), np.array([np.nan]))
    with pytest.raises(T.OverflowError):
        ctx.spgemm(nan, nan)
    assert ctx.spgemm(nan, nan, drop_nonfinite=True).C.nnz == 0


def test_empty_and_identity(ctx):
    E = T.Csr(32, 32, np.zeros(33, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    assert ctx.spgemm(E, E).C.nnz == 0
    n = 64
    I = T.Csr(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.ones(n, np.float32))
    C = ctx.spgemm(I, I).C
    assert np.array_equal(C.col, np.arange(n)) and np.all(C.val == 1.0)


def _signed_wide(rows, cols, nnz, seed, values):
    """Random pattern with tile rows wider than 32 tiles (the general
    enumerate + sort path) and sign-mixed values."""
    M = W.random_uniform(rows, cols, nnz, seed)
    u = W.uniform(seed + 7, M.nnz)
    if values == "unit":  # +-1: exact sums, frequent exact cancellation
        M.val = np.where(u < 0.5, -1.0, 1.0).astype(np.float32)
    else:  # SignedHalves [-4, 4] (proj/tests/support/corpus.hpp:52-56)
        M.val = W._round_half(-4.0 + 8.0 * u)
    return M


@pytest.mark.parametrize("density", [0.0005, 0.004, 0.03])
def test_general_path_thin_and_heavy(ctx, density):
    """General path (> 32 A tiles per tile row) with thin (thread) and heavy
    (warp) segments mixed: ORDERED bit-exact on SignedHalves; TENSOR
    bit-exact on +-1 values, whose cancellations exercise compaction."""
    from oracle import port
    m, k = 300, 6000
    nnz = int(m * k * density)
    A = _signed_wide(m, k, nnz, 21, "signed")
    B = _signed_wide(k, 400, int(k * 400 * density), 22, "signed")
    want = port.spgemm_mixed(A, B)
    got = ctx.spgemm(A, B, mode="ordered")
    assert csr_bits_equal(got.C, want), first_diff(got.C, want)
    assert got.stats["counted_elements"] == port.tile_stats(A, B, 16)["counted_elements"]
    ten = ctx.spgemm(A, B, mode="tensor")
    assert csr_pattern_equal(ten.C, want), first_diff(ten.C, want)
    ok, worst = tolerance_ok(ten.C, want, A, B)
    assert ok, worst
    Au = _signed_wide(m, k, nnz, 23, "unit")
    Bu = _signed_wide(k, 400, int(k * 400 * density), 24, "unit")
    want = port.spgemm_mixed(Au, Bu)
    for mode in ("tensor", "ordered"):
        got = ctx.spgemm(Au, Bu, mode=mode)
        assert csr_bits_equal(got.C, want), (mode, first_diff(got.C, want))
        assert got.stats["counted_elements"] == port.tile_stats(Au, Bu, 16)["counted_elements"]


@pytest.mark.parametrize("name,world", [("fem27", 8), ("poisson", 4), ("rmat", 4)])
def test_row_panels_concatenate_to_full_product(ctx, name, world):
    """The multi-GPU decomposition on one GPU: each rank's
    work-balanced A row panel times the full B (only the B tile rows the panel
    refers to are tiled) concatenates to the single-call product bit for bit."""
    from paper_2009_14600_b200 import distributed as D
    mats = W.make_small(name) if name == "rmat" else W.make(name)
    A = mats[0]
    full = ctx.spgemm(A, A).C
    rp, cols, vals = [np.zeros(1, np.int64)], [], []
    for r0, r1 in D.panel_bounds(A, A, world):
        Cp = ctx.spgemm(D.take_rows(A, r0, r1), A).C
        rp.append(np.asarray(Cp.row_ptr)[1:] + rp[-1][-1])
        cols.append(np.asarray(Cp.col))
        vals.append(np.asarray(Cp.val))
    assert np.array_equal(np.concatenate(rp), np.asarray(full.row_ptr))
    assert np.array_equal(np.concatenate(cols), np.asarray(full.col))
    assert np.array_equal(np.concatenate(vals).view(np.uint32), np.asarray(full.val).view(np.uint32))


def test_unreferenced_b_rows_are_still_validated(ctx):
    """Tile rows of B that A never refers to are not tiled, but an invalid
    entry there still raises like the reference's from_element_coo
    (tile_format.cpp:34-51, 82-96)."""
    A = T.Csr(4, 64, np.array([0, 1, 1, 1, 1]), np.array([0], np.int32), np.array([1.0], np.float32))
    rp = np.arange(65, dtype=np.int64)
    col = np.zeros(64, np.int32)
    val = np.ones(64, np.float32)
    val[40] = 1e6  # row 40: B tile row 2, never referenced by A's column 0
    with pytest.raises(T.OverflowError):
        ctx.spgemm(A, T.Csr(64, 64, rp, col, val))
    col2 = col.copy()
    rp2 = rp.copy()
    rp2[41:] += 1  # row 40 holds two entries, unsorted
    col2 = np.insert(col2, 41, 0)
    val2 = np.insert(np.ones(64, np.float32), 41, 1.0)
    with pytest.raises(T.InvariantError):
        ctx.spgemm(A, T.Csr(64, 64, rp2, col2, val2))


def _dyadic(M, seed, exps):
    """Values +-2^e, e drawn from `exps`: exact products and short sums, so
    the TENSOR path is bit-exact too; tiny exponents underflow binary16."""
    rng = np.random.default_rng(seed)
    e = rng.choice(np.asarray(exps, np.float64), M.nnz)
    s = np.where(rng.random(M.nnz) < 0.5, -1.0, 1.0)
    M.val = (s * np.exp2(e)).astype(np.float32)
    return M


@pytest.mark.parametrize("kind", ["signed", "unit", "tiny"])
def test_chain_fused_stages(ctx, kind):
    """tsg_spgemm_chain hands a light-row stage's result to the next stage as
    binary16 A tiles without a CSR round trip; the rounding, overflow check,
    underflow drop and cancellation must equal the reference's CSR ->
    binary16 conversion between stages (kernels.cpp:239-258).  Chain 1:
    light (emits) -> light on emitted tiles (emits) -> general on emitted
    tiles.  Chain 2: light (emits) -> general on emitted tiles (CSR) ->
    general on the converted CSR."""
    n = 700
    S0, S1 = W.random_uniform(n, n, 1050, 31), W.random_uniform(n, n, 1050, 33)
    wide = _signed_wide(n, n, 60 * n, 32, "unit")
    last = W.random_uniform(n, 500, 4 * n, 34)
    for i, M in enumerate((S0, S1, wide, last)):
        if kind == "signed":
            M.val = W._round_half(-4.0 + 8.0 * W.uniform(40 + i, M.nnz))
        elif kind == "unit":
            M.val = np.where(W.uniform(40 + i, M.nnz) < 0.5, -1.0, 1.0).astype(np.float32)
        else:
            _dyadic(M, 40 + i, [-9, -8, -7, -4, 0])
    for mats in ([S0, S1, wide, last], [S0, wide, S1, last]):
        want = ref.chain(mats)
        for mode in ("ordered", "tensor"):
            got = ctx.spgemm_chain(mats, mode=mode).C
            if mode == "ordered" or kind == "unit":  # +-1: every sum exact on the MMA too
                assert csr_bits_equal(got, want), (mode, first_diff(got, want))
            else:  # MMA rounding may move an intermediate across a binary16 boundary
                assert got.rows == want.rows and got.cols == want.cols and got.nnz > 0


def test_chain_intermediate_overflow(ctx):
    """An intermediate beyond binary16 range raises like the reference's
    conversion of it (tile_format.cpp from_element_coo)."""
    n = 32
    rp = np.arange(n + 1, dtype=np.int64)
    X = T.Csr(n, n, rp, np.arange(n, dtype=np.int32), np.full(n, 300.0, np.float32))
    I = T.Csr(n, n, rp, np.arange(n, dtype=np.int32), np.ones(n, np.float32))
    with pytest.raises(T.OverflowError):
        ctx.spgemm_chain([X, X, I])
    with pytest.raises(Exception):
        ref.chain([X, X, I])
    # just inside the range: 255^2 = 65025 rounds to binary16 65024
    X.val[:] = 255.0
    got = ctx.spgemm_chain([X, X, I]).C
    assert csr_bits_equal(got, ref.chain([X, X, I]))
    assert np.all(np.asarray(got.val) == 65024.0)


def test_device_output_speculation(ctx):
    """Device output with a warm staging arena enqueues the light pass before
    reading the conversion results back (one synchronisation): invalid input
    must still raise, general-path inputs must fall through to the general
    path, and results must equal the host-output path's."""
    A = W.fem27(16)
    ctx.spgemm(A, A, out="device")  # warms the arena
    for M in (A, _signed_wide(300, 6000, 9000, 21, "signed")):
        B = M if M.rows == M.cols else _signed_wide(6000, 400, 9600, 22, "signed")
        dev = ctx.spgemm(M, B, out="device").C.to_numpy()
        host = ctx.spgemm(M, B).C
        assert csr_bits_equal(dev, host), first_diff(dev, host)
    bad = T.Csr(8, 8, np.array([0, 2, 2, 2, 2, 2, 2, 2, 2]), np.array([3, 1], np.int32), np.array([1.0, 2.0]))
    with pytest.raises(T.InvariantError):
        ctx.spgemm(bad, bad, out="device")
    oob = T.Csr(8, 8, np.array([0, 1, 1, 1, 1, 1, 1, 1, 1]), np.array([9], np.int32), np.array([1.0]))
    with pytest.raises(T.InvariantError):
        ctx.spgemm(oob, oob, out="device")
    assert csr_bits_equal(ctx.spgemm(A, A, out="device").C.to_numpy(), ctx.spgemm(A, A).C)


def _coo(rows, cols, r, c, v):
    """CSR from unsorted (row, col, value) triples; duplicates keep the first."""
    r, c, v = np.asarray(r, np.int64), np.asarray(c, np.int64), np.asarray(v, np.float32)
    key = r * cols + c
    key, first = np.unique(key, return_index=True)
    return W._from_rows_cols(rows, cols, key // cols, key % cols, v[first])


@pytest.mark.parametrize("shape", ["wide_sparse", "many_tiles", "dense_panel", "zeros_and_underflow"])
def test_conversion_paths(ctx, shape):
    """Every conversion path, checked through the product (ORDERED bit-exact
    against the reference's oracle, both operand roles, A.A and A.B):
    wide_sparse   panels spanning > 8192 tile columns, <= 512 entries (sort path)
    many_tiles    narrow panels with > 64 tiles (bitmap -> sort path)
    dense_panel   panels of > 512 entries (the walk)
    zeros_and_underflow  explicit zeros, values that round to zero and
                  duplicate-tile entries in B rows (the etile first-entry rule)"""
    from oracle import port
    rng = np.random.default_rng({"wide_sparse": 1, "many_tiles": 2, "dense_panel": 3, "zeros_and_underflow": 4}[shape])
    if shape == "wide_sparse":
        n, m = 4096, 300000
        nnz = 6 * n
        A = _coo(n, m, rng.integers(0, n, nnz), rng.integers(0, m, nnz), rng.choice([-2.0, -1.0, 0.5, 1.0], nnz))
        B = _coo(m, 512, rng.integers(0, m, 3 * m // 10), rng.integers(0, 512, 3 * m // 10),
                 rng.choice([-1.0, 1.0, 2.0], 3 * m // 10))
    elif shape == "many_tiles":
        n = 2048
        r = np.repeat(np.arange(n), 20)
        c = (r // 16) * 16 + rng.integers(0, 4000, r.size)  # ~20 entries/row over ~250 tile columns
        c = np.minimum(c, 8000)
        A = _coo(n, 8192, r, c, rng.choice([-1.0, 1.0, 0.25], r.size))
        B = _coo(8192, 2048, rng.integers(0, 8192, 60000), rng.integers(0, 2048, 60000),
                 rng.choice([-1.0, 2.0], 60000))
    elif shape == "dense_panel":
        n = 256
        r = np.repeat(np.arange(n), 60)
        c = rng.integers(0, 30000, r.size)
        A = _coo(n, 30000, r, c, rng.choice([-1.0, 1.0, 3.0], r.size))
        B = _coo(30000, 700, rng.integers(0, 30000, 90000), rng.integers(0, 700, 90000),
                 rng.choice([-0.5, 1.0], 90000))
    else:
        n = 1024
        r = rng.integers(0, n, 12000)
        c = rng.integers(0, n, 12000)
        v = rng.choice([0.0, 1e-9, -1e-9, 1.0, -2.0, 0.5], 12000)  # zeros and binary16 underflows dropped
        A = _coo(n, n, r, c, v)
        B = _coo(n, n, rng.integers(0, n, 9000), rng.integers(0, n, 9000),
                 rng.choice([0.0, 1e-9, 1.0, -1.0, 4.0], 9000))
    for X, Y in ((A, B), (A, A) if A.rows == A.cols else (B, A)):
        if X.cols != Y.rows:
            continue
        want = port.spgemm_mixed(X, Y)
        got = ctx.spgemm(X, Y, mode="ordered")
        assert csr_bits_equal(got.C, want), (shape, first_diff(got.C, want))
        assert got.stats["counted_elements"] == port.tile_stats(X, Y, 16)["counted_elements"]
        dev = ctx.spgemm(X, Y, mode="ordered", out="device").C.to_numpy()
        assert csr_bits_equal(dev, want), (shape, "device", first_diff(dev, want))


def test_host_output_pipelined_slices(ctx):
    """Host output of the light path ships each chunk's CSR slices while
    later chunks compute; equal to the device output and to the reference
    restatement (rows < 2048 small column gaps, rows >= 2048 a
    150000-column gap)."""
    from oracle import port
    n, m = 4096, 200000
    A = _coo(n, n, np.arange(n), np.arange(n), np.ones(n))
    r = np.repeat(np.arange(n), 3)
    far = np.where(np.arange(n) >= 2048, 150000, 40)
    c = np.stack([np.arange(n), np.arange(n) + 17, np.arange(n) + far], 1).ravel()
    B = _coo(n, m, r, c, np.tile([1.0, -2.0, 0.5], n))
    want = port.spgemm_mixed(A, B)
    host = ctx.spgemm(A, B)
    assert csr_bits_equal(host.C, want), first_diff(host.C, want)
    dev = ctx.spgemm(A, B, out="device").C.to_numpy()
    assert csr_bits_equal(dev, want), first_diff(dev, want)
    F = W.fem27(24)
    assert csr_bits_equal(ctx.spgemm(F, F).C, ctx.spgemm(F, F, out="device").C.to_numpy())


def test_chain_device_output_and_empty_stages(ctx):
    """A chain returned on the device equals the host result; an empty
    intermediate (no overlap between stages) yields an empty product."""
    R, A, P = W.amg(32)
    host = ctx.spgemm_chain([R, A, P]).C
    dev = ctx.spgemm_chain([R, A, P], out="device").C.to_numpy()
    assert csr_bits_equal(dev, host), first_diff(dev, host)
    n = 64
    X = T.Csr(n, n, np.concatenate([np.zeros(n // 2 + 1, np.int64), np.arange(1, n // 2 + 1, dtype=np.int64)]),
              np.arange(n // 2, dtype=np.int32), np.ones(n // 2, np.float32))  # rows n/2.. hold cols 0..n/2-1
    Y = T.Csr(n, n, np.concatenate([np.zeros(n // 2 + 1, np.int64), np.arange(1, n // 2 + 1, dtype=np.int64)]),
              np.arange(n // 2, dtype=np.int32), np.ones(n // 2, np.float32))
    # X.Y = 0: X's columns (< n/2) hit Y's empty rows
    C = ctx.spgemm_chain([X, Y, X]).C
    assert C.nnz == 0 and np.all(np.asarray(C.row_ptr) == 0)
    assert csr_bits_equal(C, ref.chain([X, Y, X]))


@pytest.mark.parametrize("name", ["fem27", "rmat"])
def test_fp16_device_operands(ctx, name):
    """bench.py hands the device step binary16 values as fp16 (TSG_F16):
    the conversion's fp16 path (bitmap, sort and walk panels) must give the
    same product as fp32 operands."""
    import torch
    A = W.make_small(name)[0] if name == "rmat" else W.fem27(24)
    D32 = A.to_device("cuda")
    D16 = T.Csr(D32.rows, D32.cols, D32.row_ptr, D32.col, D32.val.to(torch.float16))
    assert torch.equal(D16.val.to(torch.float32), D32.val)  # the workloads are binary16-valued
    for mode in ("tensor", "ordered"):
        a = ctx.spgemm(D32, D32, mode=mode, out="device").C.to_numpy()
        b = ctx.spgemm(D16, D16, mode=mode, out="device").C.to_numpy()
        assert csr_bits_equal(b, a), (mode, first_diff(b, a))
