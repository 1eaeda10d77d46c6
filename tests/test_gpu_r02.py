"""GPU: round-2 contract tests -- the binary16 conversion swept through the
CUDA path, the multi-device context, malformed row pointers, device-input
stream ordering, the memory / path statistics, and the TENSOR-mode chain
bound (VERDICT r01 "parity gaps")."""
import numpy as np
import pytest

from oracle import port, ref
from paper_2009_14600_b200 import _lib as L
from paper_2009_14600_b200 import tilemul as T
from paper_2009_14600_b200 import workloads as W
from tests.helpers import csr_bits_equal, csr_pattern_equal, first_diff

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- rounding sweep
def _sweep_values():
    """Every finite binary16 value, every midpoint between neighbours, and the
    next double on both sides of each midpoint (test_half.cpp:71-89 sweep)."""
    h = np.arange(0, 0x7C00, dtype=np.uint16)  # +0 .. max finite
    pos = h.view(np.float16).astype(np.float64)
    mids = (pos[:-1] + pos[1:]) / 2.0
    lo, hi = np.nextafter(mids, -np.inf), np.nextafter(mids, np.inf)
    v = np.concatenate([pos, mids, lo, hi])
    v = np.concatenate([v, -v])
    v = v[np.abs(v) <= 65504.0]  # beyond 65504 raises (checked separately)
    return v[v != 0.0]


def _ref_round(v):
    return np.array([port.round_to_half(float(x)) for x in v])


def _diag_times_identity(ctx, vals, carrier):
    """C = D . I with D = diag(vals) in the given carrier (f64 or f32): the
    product is exactly the binary16 rounding of every diagonal value (values
    that round to zero drop, like from_element_coo)."""
    n = len(vals)
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    D = T.Csr(n, n, rp, col, vals.astype(carrier))
    I = T.Csr(n, n, rp, col, np.ones(n, np.float16))
    return ctx.spgemm(D, I, mode="ordered").C


@pytest.mark.parametrize("carrier", [np.float64, np.float32])
def test_rounding_sweep_through_conversion(ctx, carrier):
    v = _sweep_values()
    if carrier is np.float32:  # an f32 carrier holds midpoints exactly; neighbours become f32 neighbours
        v32 = v.astype(np.float32)
        v = np.unique(np.concatenate([v32, np.nextafter(v32, np.float32(np.inf)),
                                      np.nextafter(v32, np.float32(-np.inf))])).astype(np.float64)
        v = v[(np.abs(v) <= 65504.0) & (v != 0.0)]
    want = _ref_round(v)
    keep = want != 0.0
    C = _diag_times_identity(ctx, v, carrier)
    rows = np.repeat(np.arange(C.rows), np.diff(np.asarray(C.row_ptr)))
    assert np.array_equal(rows, np.nonzero(keep)[0]), "pattern: exactly the non-underflowing values survive"
    assert np.array_equal(np.asarray(C.col), rows)
    got = np.asarray(C.val, np.float32)
    assert np.array_equal(got.view(np.uint32), want[keep].astype(np.float32).view(np.uint32))


@pytest.mark.parametrize("carrier", [np.float64, np.float32])
def test_rounding_overflow_and_nonfinite(ctx, carrier):
    for x in (65504.0000001 if carrier is np.float64 else 65505.0, 65520.0, 1e6, -70000.0, np.inf, -np.inf, np.nan):
        with pytest.raises(T.OverflowError):
            _diag_times_identity(ctx, np.array([1.0, x, 2.0]), carrier)
    # drop_nonfinite drops inf / nan (but not finite overflow)
    n = 3
    rp = np.arange(n + 1, dtype=np.int64)
    D = T.Csr(n, n, rp, np.arange(n, dtype=np.int32), np.array([1.0, np.inf, np.nan]).astype(carrier))
    I = T.Csr(n, n, rp, np.arange(n, dtype=np.int32), np.ones(n, np.float16))
    C = ctx.spgemm(D, I, drop_nonfinite=True).C
    assert C.nnz == 1 and float(C.val[0]) == 1.0


# ---------------------------------------------------------------- chain bound
def _abs_chain(mats):
    """|X0| |X1| ... in float64 (dense, test sizes) -- the scale of the chain's
    rounding error."""
    acc = None
    for M in mats:
        D = np.zeros((M.rows, M.cols))
        rows = np.repeat(np.arange(M.rows), np.diff(np.asarray(M.row_ptr)))
        D[rows, np.asarray(M.col)] = np.abs(np.asarray(M.val, np.float64))
        acc = D if acc is None else acc @ D
    return acc


@pytest.mark.parametrize("kind", ["signed", "tiny"])
def test_chain_tensor_mode_bound(ctx, kind):
    """TENSOR-mode chains: pattern equal to the reference's, values within
    |c - r| <= (s * 2^-10 + 2 n 2^-23) * (|X0|...|Xn-1|)_ij, s = the number
    of binary16 roundings of intermediates (a last-bit MMA difference can
    move an intermediate across a binary16 rounding boundary: one binary16
    ulp, 2^-10 relative, per rounding).  Dyadic 'tiny' inputs: the
    binary16 roundings of intermediates make later partial sums inexact, so
    both kinds get the bound (+-1 chains are bit-exact:
    test_gpu_parity.py::test_chain_fused_stages)."""
    n = 300
    mats = [W.random_uniform(n, n, 6 * n, 51), W.random_uniform(n, n, 6 * n, 52),
            W.random_uniform(n, n, 8 * n, 53), W.random_uniform(n, 200, 4 * n, 54)]
    rng = np.random.default_rng(7)
    for M in mats:
        if kind == "signed":
            M.val = W._round_half(rng.uniform(-4.0, 4.0, M.nnz))
        else:
            e = rng.choice(np.array([-9.0, -8.0, -7.0, -4.0, 0.0]), M.nnz)
            M.val = (np.where(rng.random(M.nnz) < 0.5, -1.0, 1.0) * np.exp2(e)).astype(np.float32)
    want = ref.chain(mats)
    got = ctx.spgemm_chain(mats, mode="tensor").C
    assert csr_pattern_equal(got, want), first_diff(got, want)
    scale = _abs_chain(mats)
    rows = np.repeat(np.arange(want.rows), np.diff(want.row_ptr))
    s = len(mats) - 2
    bound = (s * 2.0 ** -10 + 2 * n * 2.0 ** -23) * scale[rows, want.col]
    err = np.abs(np.asarray(got.val, np.float64) - want.val)
    assert np.all(err <= bound), float(np.max(err / bound))


# ---------------------------------------------------------------- multi-device
def _same(a, b):
    return (np.array_equal(np.asarray(a.row_ptr), np.asarray(b.row_ptr)) and
            np.array_equal(np.asarray(a.col), np.asarray(b.col)) and
            np.array_equal(np.asarray(a.val).view(np.uint32), np.asarray(b.val).view(np.uint32)))


@pytest.mark.parametrize("k", [2, 3, 8])
def test_multi_device_context_matches_single(ctx, k):
    """tsg_create_multi with k panel workers (all on GPU 0 here; the same
    code path drives k GPUs): A split into work-balanced tile-row panels,
    the panels' CSR concatenated -- byte-identical to one context, for
    host and device operands and outputs, A.A, A.B and chains."""
    import torch
    multi = T.Context(devices=[0] * k)
    try:
        A = W.make_small("rmat")[0]
        F = W.make("poisson")[0]
        R, Am, P = W.make_small("amg")
        for (X, Y) in ((A, A), (F, F), (W.random_uniform(900, 700, 5000, 3), W.random_uniform(700, 800, 6000, 4))):
            want = ctx.spgemm(X, Y).C
            got = multi.spgemm(X, Y).C
            assert _same(got, want)
            assert len(multi.panel_ms()) == k and all(t > 0 for t in multi.panel_ms())
            got_d = multi.spgemm(X.to_device(), Y.to_device(), out="device").C
            torch.cuda.synchronize()
            assert _same(got_d.to_numpy(), want)
        want = ctx.spgemm_chain([R, Am, P]).C
        assert _same(multi.spgemm_chain([R, Am, P]).C, want)
        res = multi.spgemm(A, A)
        assert res.stats["devices"] == k
    finally:
        multi.close()


def test_multi_device_errors_propagate(ctx):
    multi = T.Context(devices=[0, 0])
    try:
        A = T.Csr(4, 4, np.array([0, 1, 2, 3, 4]), np.array([0, 1, 2, 3], np.int32),
                  np.array([1.0, 1e6, 1.0, 1.0], np.float32))
        with pytest.raises(T.OverflowError):
            multi.spgemm(A, A)
        B = T.Csr(5, 5, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
        with pytest.raises(T.DimensionError):
            multi.spgemm(A, B)
        good = W.make_small("fem27")[0]
        assert _same(multi.spgemm(good, good).C, ctx.spgemm(good, good).C)
    finally:
        multi.close()


# ---------------------------------------------------------------- malformed row_ptr
@pytest.mark.parametrize("where", ["host", "device"])
def test_malformed_row_pointers(ctx, where):
    """row_ptr[0] != 0, row_ptr[rows] != nnz, or a decreasing row_ptr raise
    InvariantError; no kernel reads entries through them (device input: the
    validation kernel gates every reader), and the context stays usable."""
    good = W.make_small("fem27")[0]
    cases = []
    rp = np.asarray(good.row_ptr).copy()
    r1 = rp.copy(); r1[-1] += 1000          # past the end of col/val
    r2 = rp.copy(); r2[0] = 5               # nonzero start
    r3 = rp.copy(); r3[10] = r3[12] + 3     # decreasing
    for bad in (r1, r2, r3):
        M = T.Csr(good.rows, good.cols, bad, good.col, good.val)
        cases.append(M.to_device() if where == "device" else M)
    for M in cases:
        with pytest.raises(T.InvariantError):
            ctx.spgemm(M, good.to_device() if where == "device" else good, out="device")
    assert _same(ctx.spgemm(good, good).C, ctx.spgemm(good, good).C)


def test_device_inputs_produced_on_torch_stream(ctx):
    """Device operands written by torch kernels immediately before the call
    (torch's current stream) are complete when the library's own stream
    reads them (tilemul._view orders the two streams)."""
    import torch
    A = W.make("fem27")[0]
    want = ctx.spgemm(A, A).C
    for _ in range(3):
        rp = torch.from_numpy(np.asarray(A.row_ptr)).cuda().to(torch.int32)  # int32 -> int64 in _view
        col = torch.from_numpy(np.asarray(A.col)).cuda()
        val = torch.from_numpy(np.asarray(A.val, np.float64)).cuda().to(torch.float16)
        got = ctx.spgemm(T.Csr(A.rows, A.cols, rp, col, val), T.Csr(A.rows, A.cols, rp, col, val), out="device").C
        assert _same(got.to_numpy(), want)


# ---------------------------------------------------------------- statistics
def test_memory_and_path_statistics(ctx):
    F = W.make("fem27")[0]
    r = ctx.spgemm(F.to_device(), F.to_device(), out="device")
    st = r.stats
    assert st["path"] == L.TSG_PATH_PANEL and st["devices"] == 1
    assert st["mem_output"] == (F.rows + 1) * 8 + st["nnz_c"] * 8
    assert st["mem_input_tiles"] > 0 and st["mem_input_elements"] > 0 and st["mem_peak"] >= st["mem_output"]
    assert st["mem_task_list"] == 0  # the light-row task list never leaves registers
    G = W.random_uniform(4000, 4000, 200_000, 9)  # > 32 tiles per tile row, ~1 entry per tile
    st = ctx.spgemm(G, G).stats
    assert st["path"] == L.TSG_PATH_GENERAL and st["mem_task_list"] > 0
    R, Am, P = W.make_small("amg")
    assert ctx.spgemm_chain([R, Am, P]).stats["path"] in (L.TSG_PATH_PANEL, L.TSG_PATH_GENERAL)


@pytest.mark.slow
def test_rmat_full_size_t16_counters(ctx):
    """R-MAT 2^20 at full size: raw / filtered pairs, segments and counted
    elements equal the T=16 restatement (oracle/tsg_oracle.c tile_stats,
    pipeline.cpp:37-109 + kernels.cpp:79-103 at T=16; ~2 min on the CPU)."""
    A = W.make("rmat")[0]
    st = ctx.spgemm(A.to_device(), A.to_device(), out="device").stats
    st16 = port.tile_stats(A, A, 16)
    for k in ("tiles_a", "raw_pairs", "filtered_pairs", "segments", "counted_elements"):
        assert st[k] == st16[k], (k, st[k], st16[k])


@pytest.mark.slow
def test_rmat_full_size_against_compiled_reference(ctx):
    """R-MAT 2^20 at full size against the compiled reference itself
    (oracle/_ref: dense_spgemm_mixed_ordered, oracle.cpp:102-121, the
    reference's bit-identical restatement of its pipeline; ~40 s on one host
    core): pattern and every fp32 value bit-equal, in both numeric modes."""
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    A = W.make("rmat")[0]
    want = ref.oracle(A)
    for mode in ("tensor", "ordered"):
        got = ctx.spgemm(A.to_device(), A.to_device(), out="device", mode=mode).C.to_numpy()
        assert csr_bits_equal(got, want), (mode, first_diff(got, want))


# ---------------------------------------------------------------- 8x8 re-tiling
def _expected_tile_vals(M, tr, tc, ei):
    """Tile element array of from_element_coo (tile_format.cpp:61-129): each
    tile's non-zero elements row-major (= bit order) from elem_index."""
    rp, col = np.asarray(M.row_ptr, np.int64), np.asarray(M.col, np.int64)
    val = np.asarray(M.val, np.float32)
    rows = np.repeat(np.arange(M.rows, dtype=np.int64), np.diff(rp))
    nz = val != 0
    rows, col, val = rows[nz], col[nz], val[nz]
    key = (rows // 8) * ((M.cols + 7) // 8) + col // 8
    order = np.lexsort(((rows % 8) * 8 + col % 8, key))
    return val[order]


@pytest.mark.parametrize("case", ["random", "odd_dims", "zeros", "rmat_slice", "empty"])
def test_tiles8_conversion_matches_reference_tiling(ctx, case):
    rng = np.random.default_rng(7)
    if case == "rmat_slice":
        M = W.rmat(14, 16, seed=3)
        M = T.Csr(M.rows, M.cols, M.row_ptr, M.col, np.asarray(M.val, np.float32) * np.float32(1.5))
    elif case == "empty":
        M = T.Csr(37, 29, np.zeros(38, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    else:
        n, m = (1000, 1000) if case != "odd_dims" else (1003, 517)
        M = ref.random_coo(11, n, m, 0.01, "signed_halves")
        val = rng.standard_normal(len(M.col)).astype(np.float32)
        if case == "zeros":  # explicit zeros are dropped, like from_element_coo
            val[rng.random(len(val)) < 0.2] = 0.0
        M = T.Csr(M.rows, M.cols, M.row_ptr, M.col, val)
    got = ctx.csr_to_tiles8(M)
    want = ref.tile8(T.Csr(M.rows, M.cols, M.row_ptr, M.col, np.asarray(M.val, np.float64)), kind="fp32")
    for k in ("tile_row", "tile_col", "bitmap", "elem_index"):
        assert np.array_equal(got[k], getattr(want, k)), k
    exp = _expected_tile_vals(M, got["tile_row"], got["tile_col"], got["elem_index"])
    assert np.array_equal(got["val"].view(np.uint32), exp.view(np.uint32))
    # round trip: tiles -> CSR on the GPU is the zero-dropped input, bit-exact
    for out in ("host", "device"):
        back = ctx.tiles8_to_csr(M.rows, M.cols, got, out=out)
        if out == "device":
            back = T.Csr(back.rows, back.cols, back.row_ptr.cpu().numpy(), back.col.cpu().numpy(),
                         back.val.cpu().numpy())
        nz = np.asarray(M.val, np.float32) != 0
        rp = np.concatenate([[0], np.cumsum(nz)])[np.asarray(M.row_ptr, np.int64)]
        assert np.array_equal(np.asarray(back.row_ptr, np.int64), rp)
        assert np.array_equal(np.asarray(back.col), np.asarray(M.col)[nz])
        assert np.array_equal(np.asarray(back.val, np.float32).view(np.uint32),
                              np.asarray(M.val, np.float32)[nz].view(np.uint32))


def test_tiles8_conversion_errors(ctx):
    M = ref.random_coo(5, 64, 64, 0.1, "signed_halves")
    val = np.asarray(M.val, np.float32).copy()
    val[3] = np.inf
    with pytest.raises(T.OverflowError):
        ctx.csr_to_tiles8(T.Csr(M.rows, M.cols, M.row_ptr, M.col, val))
    t = ctx.csr_to_tiles8(T.Csr(M.rows, M.cols, M.row_ptr, M.col, np.asarray(M.val, np.float32)))
    bad = dict(t)
    bad["tile_row"] = t["tile_row"][::-1].copy()  # unsorted tile rows
    with pytest.raises(T.InvariantError):
        ctx.tiles8_to_csr(M.rows, M.cols, bad)


# ---------------------------------------------------------------- B summaries (multi-GPU exchange)
def _as_np(bs):
    return {n: bs.arrays[n].cpu().numpy() for n in bs.arrays}


@pytest.mark.parametrize("case", ["rmat_small", "rmat14", "rect"])
def test_b_summary_matches_restatement(ctx, case):
    from paper_2009_14600_b200.tilemul import BSummary
    from paper_2009_14600_b200 import distributed as D
    from tests.helpers import bsum_reference
    B = {"rmat_small": lambda: W.make_small("rmat")[0], "rmat14": lambda: W.rmat(14, 16, seed=5),
         "rect": lambda: W.make_small("rect")[1]}[case]()
    ref = bsum_reference(B)
    whole = ctx.b_summary(B)
    got = _as_np(whole)
    assert (whole.rows, whole.tile_rows, whole.tiles, whole.nnz) == ref["dims"]
    for n in got:
        want = ref[n].view(np.int32 if ref[n].dtype == np.uint32 else np.int16)
        assert np.array_equal(got[n], want), n
    # panels summarised separately and concatenated = the whole
    parts = [ctx.b_summary(D.take_rows(B, r0, r1)) for r0, r1 in D.b_panel_bounds(B, 3)]
    cat = _as_np(BSummary.concat(parts))
    for n in got:
        assert np.array_equal(cat[n], got[n]), n
    for p in parts:
        p.free()
    whole.free()


@pytest.mark.parametrize("case", ["rmat14", "rect", "fem27_light"])
def test_spgemm_with_gathered_b_summary(ctx, case):
    """tsg_spgemm_bsum on an A panel with B's summary assembled from three row
    panels (the N-GPU exchange) equals tsg_spgemm: CSR bits and T=16 counters."""
    from paper_2009_14600_b200.tilemul import BSummary
    from paper_2009_14600_b200 import distributed as D
    if case == "rmat14":
        A = B = W.rmat(14, 16, seed=5)
    elif case == "rect":
        A, B = W.make_small("rect")
    else:
        A = B = W.make_small("fem27")[0]
    full = BSummary.concat([ctx.b_summary(D.take_rows(B, r0, r1)) for r0, r1 in D.b_panel_bounds(B, 3)])
    for r0, r1 in D.panel_bounds(A, B, 2):
        Ap = D.take_rows(A, r0, r1)
        for mode in ("tensor", "ordered"):
            want = ctx.spgemm(Ap, B, mode=mode)
            got = ctx.spgemm_bsum(Ap, B, full, mode=mode)
            assert np.array_equal(np.asarray(got.C.row_ptr), np.asarray(want.C.row_ptr))
            assert np.array_equal(np.asarray(got.C.col), np.asarray(want.C.col))
            assert np.array_equal(np.asarray(got.C.val, np.float32).view(np.uint32),
                                  np.asarray(want.C.val, np.float32).view(np.uint32))
            for k in ("raw_pairs", "filtered_pairs", "segments", "counted_elements", "nnz_c"):
                assert got.stats[k] == want.stats[k], k
            assert got.stats["path"] == want.stats["path"]


def test_b_summary_mismatch_raises(ctx):
    from paper_2009_14600_b200 import distributed as D
    A = W.rmat(12, 8, seed=2)
    part = ctx.b_summary(D.take_rows(A, 0, 1024))
    with pytest.raises(T.DimensionError):
        ctx.spgemm_bsum(A, A, part)
    part.free()


# ---------------------------------------------------------------- exact cancellation, device output
@pytest.mark.parametrize("mode", ["tensor", "ordered"])
def test_light_pass_cancellation_device_output(ctx, mode):
    """Rows whose sums cancel exactly (a B row and its negation) realise fewer
    entries than their structural count: the device-output light pass drops
    them like compact() and counted_elements stays structural."""
    rng = np.random.default_rng(3)
    n = 300
    A = ref.random_coo(21, n, n, 0.03, "signed_halves")
    rp, col = np.asarray(A.row_ptr), np.asarray(A.col)
    val = np.asarray(A.val, np.float64).copy()
    # rows 5, 17, 200: two entries k1 < k2 with B rows k1 and k2 equal up to sign
    # -> C(r, :) = a(k1) B(k1,:) + a(k2) B(k2,:) cancels where the B rows overlap
    dense = np.zeros((n, n))
    for r in range(n):
        dense[r, col[rp[r]:rp[r + 1]]] = val[rp[r]:rp[r + 1]]
    for r in (5, 17, 200):
        dense[r, :] = 0
        dense[r, 10] = 1.0
        dense[r, 11] = 1.0
    dense[11, :] = -dense[10, :]
    dense[10, 3] = 2.0
    dense[11, 3] = -2.0
    M = T.Csr(n, n, *(lambda d: (np.concatenate([[0], np.cumsum((d != 0).sum(1))]).astype(np.int64),
                               np.nonzero(d)[1].astype(np.int32), d[d != 0]))(dense))
    got = ctx.spgemm(M.to_device(), M.to_device(), mode=mode, out="device")
    want = ref.spgemm(M)  # the compiled reference: compact() drops the cancelled slots
    C = got.C.to_numpy()
    assert np.array_equal(np.asarray(C.row_ptr), want.row_ptr)
    assert np.array_equal(np.asarray(C.col), want.col)
    if mode == "ordered":
        assert np.array_equal(np.asarray(C.val, np.float32).view(np.uint32),
                              want.val.astype(np.float32).view(np.uint32))
    assert got.stats["counted_elements"] == want.counted
    assert got.stats["nnz_c"] == len(want.col) < got.stats["counted_elements"]
    assert got.stats["mem_output"] == (n + 1) * 8 + got.stats["nnz_c"] * 8
    # host output agrees
    host = ctx.spgemm(M, M, mode=mode)
    assert np.array_equal(np.asarray(host.C.col), np.asarray(C.col))


def test_tiles8_device_inputs(ctx):
    """tsg_tiles8_to_csr from device arrays (TSG_MEM_DEVICE) equals the host-input call."""
    import torch
    M = ref.random_coo(13, 700, 500, 0.02, "signed_halves")
    M = T.Csr(M.rows, M.cols, M.row_ptr, M.col, np.asarray(M.val, np.float32))
    t = ctx.csr_to_tiles8(M)
    dt = {"tile_row": torch.from_numpy(t["tile_row"].view(np.int32)).cuda(),
          "tile_col": torch.from_numpy(t["tile_col"].view(np.int32)).cuda(),
          "bitmap": torch.from_numpy(t["bitmap"].view(np.int64)).cuda(),
          "elem_index": torch.from_numpy(t["elem_index"].view(np.int64)).cuda(),
          "val": torch.from_numpy(t["val"]).cuda()}
    a = ctx.tiles8_to_csr(M.rows, M.cols, t)
    b = ctx.tiles8_to_csr(M.rows, M.cols, dt, out="device").to_numpy()
    for x, y in ((a.row_ptr, b.row_ptr), (a.col, b.col)):
        assert np.array_equal(np.asarray(x), np.asarray(y))
    assert np.array_equal(np.asarray(a.val, np.float32).view(np.uint32), np.asarray(b.val, np.float32).view(np.uint32))
    assert np.array_equal(np.asarray(a.col), np.asarray(M.col))
