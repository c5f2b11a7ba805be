"""The C-ABI library loads on a CPU-only host and exports exactly what
include/hap_b200.h declares (no compute calls here)."""
import ctypes
import os
import subprocess

import pytest

from paper_2401_05965_b200 import _lib


def test_header_declares_the_bound_functions():
    declared = set(_lib.declared_symbols())
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libhap_b200.so not built (python -m paper_2401_05965_b200.build)")
    handle = _lib.lib()
    for name in _lib.declared_symbols():
        assert isinstance(getattr(handle, name), ctypes._CFuncPtr), name
    assert handle.hap_abi_version() == 1
    assert handle.hap_nccl_version() >= 22800


def test_library_is_sm100a_only_and_uses_tensor_memory_instructions():
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "absent.so"))
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(_lib.LibraryError, match="no CPU fallback"):
        _lib.lib()
