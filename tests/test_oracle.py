"""CPU: the C restatement (oracle/tsg_oracle.c) pinned against the
reference's golden vectors (tests/golden, generated from the reference
itself) and, where it was compiled here, the reference library."""
import math

import numpy as np
import pytest

from oracle import port, ref
from tests import golden_io as G
from tests.helpers import csr_bits_equal

pytestmark = pytest.mark.skipif(not port.available(), reason="oracle/_ref/libtsg_oracle.so not built")


def test_round_to_half_probes():
    """proj/tests/test_half.cpp:36-69 cases."""
    assert port.round_to_half(1.0) == 1.0 and port.round_to_half(-2.5) == -2.5
    assert port.round_to_half(65504.0) == 65504.0
    assert port.round_to_half(2049.0) == 2048.0 and port.round_to_half(2051.0) == 2052.0
    for bad in (70000.0, -70000.0, 65504.5, math.inf, math.nan):
        with pytest.raises(port.PortError):
            port.round_to_half(bad)
    sub = 2.0 ** -24
    assert port.round_to_half(sub) == sub
    assert port.round_to_half(2.0 ** -25) == 0.0
    assert port.round_to_half(1.5 * 2.0 ** -25) == sub
    assert port.round_to_half(3.0 * 2.0 ** -25) == 2 * sub
    assert math.copysign(1, port.round_to_half(-(2.0 ** -25))) < 0
    assert math.copysign(1, port.round_to_half(-1e-12)) < 0
    assert math.copysign(1, port.round_to_half(1e-12)) > 0


def test_round_to_half_every_half():
    """test_half.cpp:71-89: every finite binary16 is a fixed point, midpoints
    tie to even, nextafter neighbours round to the nearer value."""
    halves = np.concatenate([np.arange(1024) * 2.0 ** -24] +
                            [(1024 + np.arange(1024)) * 2.0 ** (e - 25) for e in range(1, 31)])
    for i in range(0, halves.size - 1, 7):  # stride keeps the CPU suite fast
        h, nx = float(halves[i]), float(halves[i + 1])
        assert port.round_to_half(h) == h and port.round_to_half(-h) == -h
        mid = (h + nx) / 2.0
        assert port.round_to_half(mid) == (h if i % 2 == 0 else nx)
        assert port.round_to_half(np.nextafter(mid, h)) == h
        assert port.round_to_half(np.nextafter(mid, nx)) == nx


def test_round_to_half_golden():
    d = G.load("round_to_half")
    for x, y in zip(d["x"], d["y"]):
        if math.isnan(y):
            with pytest.raises(port.PortError):
                port.round_to_half(float(x))
        else:
            got = port.round_to_half(float(x))
            assert got == y and math.copysign(1, got) == math.copysign(1, y)


def test_golden_hash_of_restatement():
    """proj/tests/test_cli.cpp:149-169: FNV-1a of the oracle's .tspz."""
    d = G.load("cli_5150")
    A = G.csr(d, "A")
    C = port.spgemm_mixed(A, A)
    assert port.fnv_tiled8(C) == 0x2D882906D15D6FAF == G.expected(d, "oracle").fnv


@pytest.mark.parametrize("name", G.square_cases())
def test_mixed_oracle_matches_reference_golden(name):
    d = G.load(name)
    A = G.csr(d, "A")
    want = G.expected(d, "oracle")
    got = port.spgemm_mixed(A, A)
    assert csr_bits_equal(got, want.C), name
    assert port.fnv_tiled8(got) == want.fnv
    # the reference's 8x8 pipeline agrees with its oracle (acceptance criterion 1)
    sq = G.expected(d, "square")
    assert csr_bits_equal(sq.C, want.C)
    # tile-size-invariant totals and the T=8 counters of the reference
    st8 = port.tile_stats(A, A, 8)
    assert st8["raw_pairs"] == sq.stats["raw_pairs"]
    assert st8["filtered_pairs"] == sq.stats["filtered_pairs"]
    assert st8["segments"] == sq.stats["segments"]
    assert st8["counted_elements"] == sq.stats["counted"]
    assert port.tile_stats(A, A, 16)["counted_elements"] == sq.stats["counted"]


def test_rect_and_chain_golden():
    d = G.load("rect_small")
    A, B = G.csr(d, "A"), G.csr(d, "B")
    assert csr_bits_equal(port.spgemm_mixed(A, B), G.expected(d, "oracle").C)
    comp = G.expected(d, "compose")
    st = port.tile_stats(A, B, 8)
    assert (st["raw_pairs"], st["filtered_pairs"], st["segments"], st["counted_elements"]) == \
        (comp.stats["raw_pairs"], comp.stats["filtered_pairs"], comp.stats["segments"], comp.stats["counted"])
    d = G.load("amg_16")
    R, Am, P = G.csr(d, "R"), G.csr(d, "A"), G.csr(d, "P")
    RA = port.spgemm_mixed(R, Am)
    got = port.spgemm_mixed(RA, P)  # the restatement rounds RA to binary16 on entry
    assert csr_bits_equal(got, G.expected(d, "chain").C)


def test_cbar_matches_definition():
    d = G.load("corpus_017")
    A = G.csr(d, "A")
    colc = np.bincount(A.col, minlength=A.cols)
    rowc = np.diff(A.row_ptr)
    assert port.cbar(A, A) == int(np.dot(colc, rowc))


@pytest.mark.skipif(not ref.available(), reason="reference not compiled in this container")
def test_restatement_vs_reference_random():
    for seed in range(6):
        A = ref.random_coo(1000 + seed, 90 + 7 * seed, 90 + 7 * seed, 0.04, "wild_halves" if seed % 2 else "signed_halves")
        assert csr_bits_equal(port.spgemm_mixed(A, A), ref.oracle(A))
        r = ref.spgemm(A)
        st = port.tile_stats(A, A, 8)
        assert (st["raw_pairs"], st["filtered_pairs"], st["segments"], st["counted_elements"]) == \
            (r.raw_pairs, r.filtered_pairs, r.segments, r.counted)
