"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
header declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "elmrnn.h")).read()
    return sorted(set(re.findall(r"ELMRNN_API\s+[\w\s\*]*?\b(elmrnn_\w+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_1911_13252_b200 import build
    lib = build.build()
    syms = declared_symbols()
    assert len(syms) >= 16
    L = ctypes.CDLL(lib)
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (elmrnn_\w+)", out))
    assert exported == set(syms)
    from paper_1911_13252_b200 import elmrnn
    assert set(elmrnn.EXPORTED) == set(syms)


def test_sm100a_code_in_library():
    from paper_1911_13252_b200 import build
    lib = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1911_13252_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|orc_\w+\()", txt), f
