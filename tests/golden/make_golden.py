"""Regenerate the golden fixtures in tests/golden/ from the reference.

Runs only where the reference was compiled in place (oracle/_ref, needs
/root/reference at build time).  Every fixture's expected output comes from
the reference's own code (dense_spgemm_mixed_ordered, spgemm_square, the
pass composition, round_to_half) -- never from this repo's CUDA path or the
C restatement -- following the reference's rule that golden files come from
the oracle (proj/tests/test_cli.cpp:149-169).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from paper_2009_14600_b200 import workloads as W  # noqa: E402
from paper_2009_14600_b200.tilemul import Csr  # noqa: E402


def pack(prefix: str, M) -> dict:
    return {f"{prefix}_shape": np.array([M.rows, M.cols], np.int64), f"{prefix}_rp": np.asarray(M.row_ptr, np.int64),
            f"{prefix}_col": np.asarray(M.col, np.int32), f"{prefix}_val": np.asarray(M.val, np.float64)}


def result(prefix: str, r) -> dict:
    d = pack(prefix, Csr(r.rows, r.cols, r.row_ptr, r.col, r.val))
    d[f"{prefix}_stats"] = np.array([r.raw_pairs, r.filtered_pairs, r.segments, r.counted, r.realized], np.uint64)
    d[f"{prefix}_fnv"] = np.array([r.fnv], np.uint64)
    d[f"{prefix}_tiles"] = np.stack([r.tile_row.astype(np.uint64), r.tile_col.astype(np.uint64), r.bitmap,
                                     r.elem_index]) if r.tile_row.size else np.zeros((4, 0), np.uint64)
    return d


def square_case(name: str, A, note: str):
    d = {"note": np.array(note)}
    d.update(pack("A", A))
    d.update(result("oracle", ref.oracle(A)))         # dense_spgemm_mixed_ordered
    d.update(result("square", ref.spgemm(A)))         # spgemm_square (8x8 pipeline)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)


def main():
    # proj/tests/test_cli.cpp:149-169: seed 5150, 120^2, 5%, SignedHalves
    square_case("cli_5150", ref.random_coo(5150, 120, 120, 0.05), "golden FNV-1a 0x2d882906d15d6faf")
    # proj/tests/acceptance.cpp:45-58 corpus members
    for i in (0, 17, 58, 133, 199):
        square_case(f"corpus_{i:03d}", ref.corpus("main", i), f"acceptance corpus matrix {i}")
    # proj/tests/test_kernels.cpp:332-348 WildHalves odd-dims corpus
    for i in (0, 11):
        square_case(f"wild_{i:02d}", ref.corpus("wild", i), f"WildHalves corpus matrix {i}")
    # cancellation fixtures, proj/tests/acceptance.cpp:62-98
    m1 = Csr(16, 16, np.array([0, 2, 3, 4] + [4] * 13, np.int64), np.array([1, 2, 8, 8], np.int32),
             np.array([1.0, -1.0, 5.0, 5.0]))
    square_case("cancel_1", m1, "acceptance.cpp:66-71")
    rows, cols, vals = [], [], []
    for j in range(8):
        rows += [0, 0, 2 * j, 2 * j + 1]
        cols += [2 * j, 2 * j + 1, 17, 17]
        vals += [3.0, -3.0, 0.25, 0.25]
    order = np.lexsort((cols, rows))
    r, c, v = np.array(rows)[order], np.array(cols)[order], np.array(vals)[order]
    rp = np.zeros(33, np.int64)
    rp[1:] = np.cumsum(np.bincount(r, minlength=32))
    square_case("cancel_2", Csr(32, 32, rp, c.astype(np.int32), v), "acceptance.cpp:72-82")
    # pattern / positive values (acceptance criteria 5 / 6 value modes)
    square_case("pattern_64", ref.random_coo(223, 64, 64, 0.05, "pattern"), "Pattern matrix")
    square_case("posreal_64", ref.random_coo(311, 64, 64, 0.08, "positive_reals"), "PositiveReals (rounded)")
    # the BASELINE configs at test size
    square_case("poisson_32", W.poisson2d(32), "2D 5-point Poisson 32x32")
    square_case("fem27_8", W.fem27(8), "27-point stencil 8^3")
    A = W.random_uniform(3000, 1500, 6000, 5)
    B = W.random_uniform(1500, 3000, 6000, 6)
    d = {"note": np.array("rect A.B, pass composition")}
    d.update(pack("A", A))
    d.update(pack("B", B))
    d.update(result("oracle", ref.oracle(A, B)))
    d.update(result("compose", ref.spgemm(A, B)))
    np.savez_compressed(os.path.join(HERE, "rect_small.npz"), **d)
    R, Am, P = W.amg(16)
    d = {"note": np.array("AMG (R.A).P 16^3 -> 8^3 with binary16 downcast")}
    d.update(pack("R", R))
    d.update(pack("A", Am))
    d.update(pack("P", P))
    d.update(result("chain", ref.chain([R, Am, P])))
    np.savez_compressed(os.path.join(HERE, "amg_16.npz"), **d)
    # round_to_half (proj/src/half.cpp:12-36) on the test_half.cpp probes
    xs = [1.0, 0.0, -2.5, 65504.0, 2049.0, -2049.0, 2051.0, 2.0 ** -24, 2.0 ** -25, 1.5 * 2.0 ** -25,
          3.0 * 2.0 ** -25, -(2.0 ** -25), -1e-12, 1e-12, 0.1, 1.0 / 3.0, 65519.0]
    rng = np.random.default_rng(7)
    xs += list(rng.uniform(-65504, 65504, 4000)) + list(np.ldexp(rng.uniform(1, 2, 4000), rng.integers(-30, 16, 4000)))
    def r2h(x):  # NaN marks OverflowError (status 3)
        try:
            return ref.round_to_half(x)
        except ref.RefError as e:
            assert e.status == 3
            return float("nan")
    ys = np.array([r2h(x) for x in xs])
    np.savez_compressed(os.path.join(HERE, "round_to_half.npz"), x=np.array(xs), y=ys)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
