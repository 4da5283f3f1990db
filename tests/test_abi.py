"""CPU checks of the boundary: the library builds for sm_100a, loads, and exports
every symbol include/*.h declares (no compute calls without a GPU)."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(b200_\w+)\s*\(", txt))
    return sorted(names)


@pytest.fixture(scope="module")
def libpath():
    from paper_2409_08729_b200 import _build
    return _build.build()


def test_header_declares_entry_points():
    names = _declared()
    for must in ("b200_log_iv_f64", "b200_log_kv_f64", "b200_vmf_fit_f32", "b200_vmf_colsum_f32",
                 "b200_vmf_fit_from_colsum"):
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (b200_\w+)", out))
    assert set(_declared()) <= exported


def test_binding_signatures_cover_header():
    from paper_2409_08729_b200 import _lib
    assert set(_declared()) == set(_lib.SIGNATURES)


def test_built_for_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_import_in_product():
    for f in glob.glob(os.path.join(ROOT, "paper_2409_08729_b200", "**", "*.py"), recursive=True):
        src = open(f).read()
        assert not re.search(r"^\s*(import oracle|from oracle)", src, re.M), f


def test_argument_errors_without_gpu(libpath):
    """Invalid arguments are rejected before any CUDA call (works with no device)."""
    import paper_2409_08729_b200 as B
    L = B.lib()
    assert L.b200_log_iv_f64(None, None, None, -1, None) == 1
    assert L.b200_log_iv_f64(None, None, None, 0, None) == 0
    assert L.b200_log_kv_f64(None, None, None, 5, None) == 1
    assert b"null" in L.b200_last_error()
