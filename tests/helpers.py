"""Comparison helpers shared by the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np


def csr_pattern_equal(C, R) -> bool:
    return (C.rows == R.rows and C.cols == R.cols and np.array_equal(np.asarray(C.row_ptr), R.row_ptr)
            and np.array_equal(np.asarray(C.col), R.col))


def csr_bits_equal(C, R) -> bool:
    """Positions and fp32 bit patterns equal (bit_equal_coo, corpus.hpp:102-116)."""
    if not csr_pattern_equal(C, R):
        return False
    a = np.asarray(C.val, dtype=np.float32).view(np.uint32)
    b = np.asarray(R.val, dtype=np.float64).astype(np.float32).view(np.uint32)
    return np.array_equal(a, b)


def first_diff(C, R) -> str:
    if C.rows != R.rows or C.cols != R.cols:
        return f"dims {C.rows}x{C.cols} vs {R.rows}x{R.cols}"
    rp = np.asarray(C.row_ptr)
    if not np.array_equal(rp, R.row_ptr):
        i = int(np.nonzero(rp != R.row_ptr)[0][0])
        return f"row_ptr[{i}] {rp[i]} vs {R.row_ptr[i]} (nnz {rp[-1]} vs {R.row_ptr[-1]})"
    col = np.asarray(C.col)
    if not np.array_equal(col, R.col):
        i = int(np.nonzero(col != R.col)[0][0])
        return f"col[{i}] {col[i]} vs {R.col[i]}"
    a = np.asarray(C.val, dtype=np.float32)
    b = R.val.astype(np.float32)
    i = np.nonzero(a.view(np.uint32) != b.view(np.uint32))[0]
    return f"{i.size} value bit mismatches, first at {int(i[0])}: {a[i[0]]!r} vs {b[i[0]]!r}" if i.size else "equal"


def tolerance_ok(C, R, A, B, factor: float = 2.0, rel: float = 0.0) -> tuple[bool, float]:
    """|c - r| <= factor * n * 2^-23 * sum_k |a_ik b_kj| + rel * |r|.

    The first term is the SURVEY.md 8(d) bound for well-scaled inputs.  `rel`
    is the measured allowance for TENSOR mode on inputs spanning the whole
    binary16 range (WildHalves): the MMA aligns each 16-wide k block to its
    largest exponent, products with a zero factor included, so small terms
    keep fewer bits (scripts/tc_worst_element.py, numerics).
    Needs the |A|.|B| product and per-element product counts; computed with
    a float64 Gustavson over the same CSR (test sizes only)."""
    absprod, nprod = _abs_product(A, B)
    rows = np.repeat(np.arange(R.rows), np.diff(R.row_ptr))
    key = rows.astype(np.int64) * R.cols + R.col
    bound = np.array([factor * nprod.get(k, 1) * 2.0 ** -23 * absprod.get(k, 0.0) for k in key.tolist()])
    bound = bound + rel * np.abs(np.asarray(R.val, np.float64))
    err = np.abs(np.asarray(C.val, np.float64) - R.val)
    return bool(np.all(err <= bound)), float(np.max(err / np.maximum(bound, 1e-300))) if err.size else 0.0


def _abs_product(A, B):
    absprod, nprod = {}, {}
    arp, acol, aval = np.asarray(A.row_ptr), np.asarray(A.col), np.abs(np.asarray(A.val, np.float64))
    brp, bcol, bval = np.asarray(B.row_ptr), np.asarray(B.col), np.abs(np.asarray(B.val, np.float64))
    aval = aval.astype(np.float16).astype(np.float64)
    bval = bval.astype(np.float16).astype(np.float64)
    for i in range(A.rows):
        for p in range(arp[i], arp[i + 1]):
            k = acol[p]
            for q in range(brp[k], brp[k + 1]):
                key = i * B.cols + int(bcol[q])
                absprod[key] = absprod.get(key, 0.0) + aval[p] * bval[q]
                nprod[key] = nprod.get(key, 0) + 1
    return absprod, nprod


def quadrants(tiles) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """16x16 tiles -> the 8x8 tiles they contain (SURVEY.md 8(c) bridge):
    tile (I,J) quadrant (qr,qc) -> 8x8 tile (2I+qr, 2J+qc), bit 8r+c =
    mask bit 16(8qr+r)+(8qc+c); empty quadrants dropped; sorted (row, col)."""
    rows, cols, bms = [], [], []
    m = tiles.row_masks.astype(np.uint64)
    for qr in (0, 1):
        for qc in (0, 1):
            bm = np.zeros(m.shape[0], dtype=np.uint64)
            for r in range(8):
                byte = (m[:, 8 * qr + r] >> np.uint64(8 * qc)) & np.uint64(0xFF)
                bm |= byte << np.uint64(8 * r)
            keep = bm != 0
            rows.append(2 * tiles.tile_row[keep].astype(np.int64) + qr)
            cols.append(2 * tiles.tile_col[keep].astype(np.int64) + qc)
            bms.append(bm[keep])
    rows, cols, bms = np.concatenate(rows), np.concatenate(cols), np.concatenate(bms)
    order = np.lexsort((cols, rows))
    return rows[order], cols[order], bms[order]


def bsum_reference(M) -> dict:
    """numpy restatement of tsg_bsum for a CSR whose values are binary16
    (tsparse_b200.h): per row the distinct 16-column tiles it touches, per
    16-row tile row its tile count and occupied rows (| 1 << 16 when every
    tile occupies one row), per tile (tile row, then column order) its row
    occupancy, per entry its tile's rank in the tile row (| 0x80000000 unless
    the first of that tile in its row) and its binary16 bits."""
    rp = np.asarray(M.row_ptr, np.int64)
    col = np.asarray(M.col, np.int64)
    h16 = np.asarray(M.val, np.float64).astype(np.float16).view(np.uint16)
    rows = M.rows
    tr = (rows + 15) // 16
    row_of = np.repeat(np.arange(rows, dtype=np.int64), np.diff(rp))
    kept = (h16 & 0x7FFF) != 0
    J = col >> 4
    T = row_of >> 4
    # tiles: distinct (tile row, J) among kept entries, sorted
    key = T[kept] * (1 << 32) + J[kept]
    tiles, inv = np.unique(key, return_inverse=True)
    tile_T = tiles >> 32
    tile_count = np.bincount(tile_T, minlength=tr).astype(np.uint32)
    first = np.concatenate([[0], np.cumsum(tile_count)])[:-1]
    rank = np.arange(len(tiles), dtype=np.int64) - first[tile_T]
    ro = np.zeros(len(tiles), np.int64)
    np.bitwise_or.at(ro, inv, 1 << (row_of[kept] & 15))
    rinfo = np.zeros(tr, np.int64)
    np.bitwise_or.at(rinfo, tile_T, ro)
    single = np.ones(tr, bool)
    multi = np.array([bin(int(x)).count("1") > 1 for x in ro], bool)
    single[np.unique(tile_T[multi])] = False
    rinfo = rinfo | np.where(single, 1 << 16, 0)
    etile = np.full(len(col), 0xFFFFFFFF, np.uint64)
    et = rank[inv].astype(np.uint64)
    # dup: not the first kept entry of its (row, tile)
    kr, kj = row_of[kept], J[kept]
    dup = np.zeros(len(kr), bool)
    dup[1:] = (kr[1:] == kr[:-1]) & (kj[1:] == kj[:-1])
    etile[kept] = et | np.where(dup, 0x80000000, 0).astype(np.uint64)
    njt = np.bincount(kr[~dup], minlength=rows).astype(np.uint32)
    return {"njt": njt, "tile_count": tile_count, "rinfo": rinfo.astype(np.uint32), "ro": ro.astype(np.uint16),
            "etile": etile.astype(np.uint32), "h16": np.where(kept, h16, 0).astype(np.uint16),
            "dims": (rows, tr, len(tiles), len(col))}
