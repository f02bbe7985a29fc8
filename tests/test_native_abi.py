"""CPU checks of the C-ABI boundary: both libraries load and export every symbol the
include/*.h headers declare (no device compute is called here)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header: str) -> list[str]:
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", text)))


def test_host_library_exports_header():
    from paper_2602_05754_b200 import _native

    lib = _native.host()
    names = declared("pipefreeze_c.h")
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_device_library_exports_header():
    pytest.importorskip("torch")
    from paper_2602_05754_b200 import _native

    lib = _native.device()
    names = declared("pf_device.h")
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2602_05754_b200 import _native

    monkeypatch.setattr(_native, "LIB_DIR", str(tmp_path))
    with pytest.raises(_native.NativeLibraryError):
        _native._load("libpf_device.so")
