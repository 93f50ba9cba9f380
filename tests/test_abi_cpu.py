"""CPU-only checks of the product boundary (no GPU; no compute calls).

* libisax.so loads and exports every function include/isax.h declares.
* The product's breakpoint table (csrc/breakpoints.inc, produced by its own generator) equals
  the oracle's table, which is computed independently with mpmath.
* The product package never imports the oracle.
"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "isax.h")
LIB = os.path.join(ROOT, "paper_2009_01614_b200", "libisax.so")


def declared_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(isax_[a-z_0-9]+)\s*\(", txt, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ("isax_build", "isax_nn1", "isax_free", "isax_last_error"):
        assert must in names
    assert len(names) >= 10


@pytest.mark.skipif(not os.path.exists(LIB), reason="libisax.so not built")
def test_library_loads_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared_functions():
        assert hasattr(lib, name), name
    lib.isax_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.isax_version()


@pytest.mark.skipif(not os.path.exists(LIB), reason="libisax.so not built")
def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_breakpoints_equal_oracle_table():
    from oracle.breakpoints import breakpoints

    txt = open(os.path.join(ROOT, "paper_2009_01614_b200", "csrc", "breakpoints.inc")).read()
    body = txt[txt.index("ISAX_BETA_INIT") :]
    vals = [float.fromhex(v) for v in re.findall(r"-?0x[0-9a-fA-F.]+p[+-]\d+", body)]
    assert vals == list(breakpoints(256))


def test_product_generator_reproduces_committed_table():
    from paper_2009_01614_b200.tools import gen_breakpoints

    from oracle.breakpoints import breakpoints

    assert gen_breakpoints.table(16) == list(breakpoints(16))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2009_01614_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".inc")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f
                assert "liboracle" not in src, f
