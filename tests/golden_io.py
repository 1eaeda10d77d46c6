"""Load the committed golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the reference itself)."""
from __future__ import annotations

import glob
import os
from dataclasses import dataclass

import numpy as np

from paper_2009_14600_b200.tilemul import Csr

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Expected:
    C: Csr            # float64 carrier of the reference's fp32 values
    stats: dict       # reference T=8 counters (zeros for the element oracle)
    fnv: int          # FNV-1a of the .tspz serialisation (0 if not recorded)
    tiles: np.ndarray  # (4, ntiles): tile_row, tile_col, bitmap, elem_index (8x8)


def csr(d, prefix: str) -> Csr:
    rows, cols = (int(x) for x in d[f"{prefix}_shape"])
    return Csr(rows, cols, d[f"{prefix}_rp"], d[f"{prefix}_col"], d[f"{prefix}_val"])


def expected(d, prefix: str) -> Expected:
    st = d[f"{prefix}_stats"]
    keys = ("raw_pairs", "filtered_pairs", "segments", "counted", "realized")
    return Expected(csr(d, prefix), {k: int(v) for k, v in zip(keys, st)}, int(d[f"{prefix}_fnv"][0]),
                    d[f"{prefix}_tiles"])


def load(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def square_cases() -> list[str]:
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        n = os.path.basename(p)[:-4]
        if "square_shape" in np.load(p).files:
            out.append(n)
    return out
