"""The GPU-backed front end tools/tilemul_gpu (the reference's CLI,
proj/tools/tilemul.cpp) and the file formats it shares with the reference:
.tspz (tiled_io.cpp) and Matrix Market (mm_io.cpp).

CPU tests run every path that does not multiply (convert, stats, error exit
codes); GPU tests run square / compare / bench and the reference's own
acceptance gates with TILEMUL_BIN pointed at tools/tilemul_gpu."""
import os
import subprocess

import numpy as np
import pytest

from oracle import port
from tests import golden_io as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "tilemul_gpu")
ACCEPTANCE = os.path.join(ROOT, "oracle", "_ref", "acceptance")
GOLDEN_FNV = 0x2D882906D15D6FAF  # proj/tests/test_cli.cpp:149-169

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="tools/tilemul_gpu not built")


def fnv1a(b: bytes) -> int:
    h = 1469598103934665603
    for c in b:
        h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def write_mtx(path, M):
    rp, col, val = (np.asarray(x) for x in (M.row_ptr, M.col, M.val))
    rows = np.repeat(np.arange(M.rows), np.diff(rp))
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{M.rows} {M.cols} {len(col)}\n")
        for r, c, v in zip(rows, col, val):
            f.write(f"{r + 1} {c + 1} {float(v)!r}\n")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_convert_reproduces_reference_golden_hash(tmp_path):
    """from_element_coo(oracle C, Fp32Stored) -> .tspz: the reference's
    golden bytes (the oracle half of test_cli.cpp:149-169)."""
    d = G.load("cli_5150")
    C = port.spgemm_mixed(G.csr(d, "A"), G.csr(d, "A"))
    write_mtx(tmp_path / "c.mtx", C)
    r = run("convert", "--input", str(tmp_path / "c.mtx"), "--output", str(tmp_path / "c.tspz"),
            "--precision", "fp32")
    assert r.returncode == 0, r.stderr
    assert fnv1a((tmp_path / "c.tspz").read_bytes()) == GOLDEN_FNV


def test_convert_fp16_layout(tmp_path):
    d = G.load("cli_5150")
    A = G.csr(d, "A")
    write_mtx(tmp_path / "a.mtx", A)
    assert run("convert", "--input", str(tmp_path / "a.mtx"), "--output", str(tmp_path / "a.tspz")).returncode == 0
    b = (tmp_path / "a.tspz").read_bytes()
    assert b[:4] == b"TSPZ" and int.from_bytes(b[4:8], "little") == 1 and b[8] == 0  # fp16 kind
    rows, cols, nt, ne = (int.from_bytes(b[9 + 8 * i:17 + 8 * i], "little") for i in range(4))
    assert (rows, cols, ne) == (A.rows, A.cols, A.nnz)
    assert len(b) == 41 + nt * 24 + ne * 2


def test_stats_matches_reference_counters(tmp_path):
    d = G.load("cli_5150")
    A = G.csr(d, "A")
    write_mtx(tmp_path / "a.mtx", A)
    r = run("stats", "--input", str(tmp_path / "a.mtx"), "--json")
    assert r.returncode == 0, r.stderr
    import json
    s = json.loads(r.stdout)
    st8 = port.tile_stats(A, A, 8)
    assert s["nnzA"] == A.nnz and s["nnzCbar"] == port.cbar(A, A)
    assert s["nnzCbarTilesRaw"] == st8["raw_pairs"] and s["nnzCbarTilesFiltered"] == st8["filtered_pairs"]


def _advise_rules(s: dict, raw: bool) -> dict:
    """advise (analytics.cpp:93-118): the published thresholds on the stats."""
    pairs = s["nnzCbarTilesRaw"] if raw else s["nnzCbarTilesFiltered"]
    ratio = s["nnzCbar"] / pairs if pairs else 0.0
    nnz, avg = s["nnzA"], s["avgRow"]
    return {"cuSPARSE": nnz > 200000, "CUSP": ratio >= 1.0, "RMerge2": avg > 42 and nnz > 100000,
            "Nsparse": avg > 42 and nnz > 100000, "AC-SpGEMM": ratio > 9.0, "spECK": avg > 42 and nnz > 300000,
            "global": nnz > 300000 and avg > 42, "globalRelaxed": nnz > 300000 and avg > 21}


@pytest.mark.parametrize("raw", [False, True])
def test_advise_evaluates_thresholds_on_stats(tmp_path, raw):
    """`advise --json` (tilemul.cpp:146-162): the eight approaches in the
    reference's order with their conditions, recommended per the thresholds
    on the same statistics `stats` prints."""
    import json
    d = G.load("cli_5150")
    A = G.csr(d, "A")
    write_mtx(tmp_path / "a.mtx", A)
    s = json.loads(run("stats", "--input", str(tmp_path / "a.mtx"), "--json").stdout)
    args = ["advise", "--input", str(tmp_path / "a.mtx"), "--json"] + (["--raw-tile-ratio"] if raw else [])
    r = run(*args)
    assert r.returncode == 0, r.stderr
    adv = json.loads(r.stdout)
    want = _advise_rules(s, raw)
    assert [e["approach"] for e in adv] == list(want)
    assert {e["approach"]: e["recommended"] for e in adv} == want
    assert all(e["condition"] for e in adv)
    table = run("advise", "--input", str(tmp_path / "a.mtx")).stdout.splitlines()
    assert table[0].startswith("approach") and len(table) == 9


def test_exit_codes(tmp_path):
    """tilemul.cpp:285-306 / acceptance criterion 10 (acceptance.cpp:489-515)."""
    (tmp_path / "bad.mtx").write_text("not a banner\n")
    assert run("stats", "--input", str(tmp_path / "bad.mtx")).returncode == 2
    (tmp_path / "big.mtx").write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e6\n")
    assert run("convert", "--input", str(tmp_path / "big.mtx"), "--output", str(tmp_path / "b.tspz")).returncode == 3
    (tmp_path / "rect.mtx").write_text("%%MatrixMarket matrix coordinate real general\n4 8 1\n1 1 1\n")
    assert run("square", "--input", str(tmp_path / "rect.mtx"), "--output", str(tmp_path / "c.tspz")).returncode == 4
    (tmp_path / "trunc.tspz").write_bytes(b"TSPZ\x01\x00\x00\x00")
    assert run("stats", "--input", str(tmp_path / "trunc.tspz")).returncode == 2
    assert run("square", "--bogus").returncode == 1


@pytest.mark.gpu
def test_square_and_bench_reproduce_golden_bytes(tmp_path):
    """The GPU front end's `square` (default ordered numerics) writes the
    reference's golden .tspz; `bench` reports the same FNV-1a hash."""
    d = G.load("cli_5150")
    write_mtx(tmp_path / "a.mtx", G.csr(d, "A"))
    r = run("square", "--input", str(tmp_path / "a.mtx"), "--output", str(tmp_path / "c.tspz"),
            "--report", str(tmp_path / "r.json"))
    assert r.returncode == 0, r.stderr
    assert fnv1a((tmp_path / "c.tspz").read_bytes()) == GOLDEN_FNV
    import json
    rep = json.loads((tmp_path / "r.json").read_text())
    assert rep["nnzC"] == G.expected(d, "oracle").C.nnz and rep["smapeVsFp64"] < 0.1
    b = run("bench", "--input", str(tmp_path / "a.mtx"), "--iters", "3")
    assert b.returncode == 0, b.stderr
    assert int(b.stdout.strip().splitlines()[1].split(",")[-1]) == GOLDEN_FNV
    t = run("square", "--input", str(tmp_path / "a.mtx"), "--output", str(tmp_path / "t.tspz"), "--numerics", "tensor")
    assert t.returncode == 0, t.stderr
    c = run("compare", "--input", str(tmp_path / "a.mtx"), "--mode", "mixed")
    assert c.returncode == 0 and "SMAPE vs mixed oracle: 0 %" in c.stdout, c.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(ACCEPTANCE), reason="reference acceptance binary not built")
def test_reference_acceptance_against_gpu_cli(tmp_path):
    """The reference's acceptance binary, unmodified, with TILEMUL_BIN pointed at
    the GPU front end: criteria 7 (square determinism) and 10 (round trip and
    exit codes) exercise tools/tilemul_gpu; the rest check the reference itself."""
    env = dict(os.environ, TILEMUL_BIN=CLI)
    r = subprocess.run([ACCEPTANCE], capture_output=True, text=True, timeout=900, env=env, cwd=tmp_path)
    lines = r.stdout.splitlines()
    for c in (7, 10):
        assert any(ln.startswith("PASS") and f"criterion {c}:" in ln for ln in lines), r.stdout
    assert not any(ln.startswith("FAIL") for ln in lines), r.stdout
