"""CPU: the C-ABI library loads, exports every symbol include/tsparse_b200.h
declares, and the ctypes mirror matches the header's struct layouts.  No
compute call is made (there is no GPU here)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2009_14600_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tsparse_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^TSG_API\s+(?:const\s+)?\w+\s*\*?\s*(tsg_\w+)\s*\(", src, re.M)))


def test_header_declares_what_binding_expects():
    assert sorted(L.EXPORTS) == declared()


def test_library_exports_every_symbol():
    lib = L.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.tsg_abi_version() == 4


def test_library_has_no_cpu_fallback_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    ours = {s for s in exported if "tsg" in s}  # the static cudart keeps its own exports
    assert ours == set(declared())


@pytest.mark.skipif(subprocess.run(["which", "gcc"], capture_output=True).returncode != 0, reason="no gcc")
def test_struct_layouts_match_header():
    structs = {"tsg_csr": L.tsg_csr, "tsg_csr_out": L.tsg_csr_out, "tsg_tiles_out": L.tsg_tiles_out,
               "tsg_options": L.tsg_options, "tsg_run_stats": L.tsg_run_stats, "tsg_tiles8": L.tsg_tiles8,
               "tsg_tiles8_out": L.tsg_tiles8_out, "tsg_bsum": L.tsg_bsum}
    prog = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){"]
    for s, cls in structs.items():
        prog.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f, _ in cls._fields_:
            prog.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    prog.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write("\n".join(prog))
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-o", exe, c], check=True)
        got = dict(l.split() for l in subprocess.run([exe], capture_output=True, text=True).stdout.splitlines())
    for s, cls in structs.items():
        assert int(got[s]) == C.sizeof(cls), s
        for f, _ in cls._fields_:
            assert int(got[f"{s}.{f}"]) == getattr(cls, f).offset, f"{s}.{f}"
