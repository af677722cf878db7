"""The C-ABI library loads and exports every entry point include/t2s2.h
declares (no GPU needed: nothing is called)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "t2s2.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void\*?|const char\*)\s+(t2s2_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    for required in ("t2s2_round", "t2s2_solve", "t2s2_march", "t2s2_apply", "t2s2_norm"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2506_04732_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.fail(f"{_native.LIB_PATH} not built (run make)")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(_native.EXPORTED)


def test_library_is_sm100a():
    import subprocess

    from paper_2506_04732_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout
