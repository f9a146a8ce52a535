"""C-ABI boundary (CPU-only checks): the in-tree library loads and exports every entry
point declared in include/nlrom_b200.h; no compute calls (no GPU here)."""

import ctypes
import os
import re

import pytest

from paper_2102_11026_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "nlrom_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nlrom_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_binding_surface():
    syms = declared_symbols()
    assert set(syms) == set(_lib.EXPORTED), set(syms) ^ set(_lib.EXPORTED)


@pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="library not built (run __graft_entry__.build())")
def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(L, s), s
    _lib.lib()   # argtypes / restype binding works


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()
