"""The C-ABI library loads and exports every symbol include/pf_b200.h declares (no GPU calls)."""

import ctypes
import os
import re

from paper_2209_07969_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pf_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding_table():
    assert set(header_symbols()) == set(_native.EXPORTED)


def test_library_exports_all_symbols():
    lib = _native.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.pf_version()


def test_struct_layouts_match_header():
    # sizes of the C structs as laid out by the x86-64 SysV ABI
    assert ctypes.sizeof(_native.PfMesh) == 4 * 2 + 8 * 2 + 8 * 6 + 4 * 3 + 4 + 8 * 3
    assert ctypes.sizeof(_native.PfMaterial) == 8 * 8 + 8
    assert ctypes.sizeof(_native.PfConfig) == 8 * 4 + 4 * 2 + 8 + 8
