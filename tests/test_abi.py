"""C-ABI boundary checks that need no GPU (-m "not gpu"): the library loads, it
exports every entry point include/piko.h declares, and host-side argument
validation rejects bad shapes before touching CUDA."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "piko.h")


@pytest.fixture(scope="module")
def piko():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1404_6293_b200 as p
    return p


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(piko_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("piko_create", "piko_draw", "piko_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol(piko):
    names = declared_functions()
    lib = ctypes.CDLL(piko.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(piko.EXPORTS) == names
    out = subprocess.check_output(["nm", "-D", "--defined-only", piko.LIB_PATH], text=True)
    exported = set(re.findall(r" T (piko_[a-z0-9_]+)$", out, flags=re.M))
    assert set(names) <= exported


def test_library_is_sm100a(piko):
    out = subprocess.check_output(["cuobjdump", "--list-elf", piko.LIB_PATH], text=True)
    assert "sm_100a" in out


@pytest.mark.parametrize("W,H,bw,bh", [(0, 64, 8, 8), (64, 0, 8, 8), (16385, 64, 8, 8),
                                       (64, 64, 4, 8), (64, 64, 12, 8), (64, 64, 8, 128),
                                       (64, 64, 0, 0)])
def test_create_rejects_bad_arguments(piko, W, H, bw, bh):
    h = piko.lib.piko_create(W, H, bw, bh)
    assert not h
    assert piko.lib.piko_last_error(None)


def test_null_safe_destroy_and_errors(piko):
    piko.lib.piko_destroy(None)
    assert piko.lib.piko_draw(None, None, None, 0, None, None, None, None, None) == piko.PIKO_EINVAL
    assert piko.lib.piko_finish(None) == piko.PIKO_EINVAL


def test_product_package_never_imports_oracle():
    """The product path must not route through the oracle."""
    pkg = os.path.join(ROOT, "paper_1404_6293_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace(
                    "oracle/piko_oracle.c", ""), f
