"""CPU tests of the C-ABI boundary: the library builds, loads without a GPU,
and exports exactly the entry points include/vsb200.h declares."""

from __future__ import annotations

import ctypes
import re
import subprocess

import pytest

from paper_1805_03709_b200 import _lib, build


def header_functions() -> set[str]:
    text = _lib.HEADER_PATH.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(vs_[a-z0-9_]+)\s*\(", text))


def test_library_builds_and_loads():
    path = build.build()
    assert path.exists()
    lib = _lib.load()
    assert lib.vs_abi_version() == 2


def test_every_header_symbol_is_exported_and_bound():
    declared = header_functions()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (vs_[a-z0-9_]+)", out))
    assert declared <= exported, declared - exported
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    lib = _lib.load()
    for name in declared:
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_no_host_symbols_leak_beyond_the_abi():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    vs = set(re.findall(r"\bT (vs_[a-z0-9_]+)", out))
    assert vs == header_functions()


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_map_to_valueerror_without_gpu():
    lib = _lib.load()
    h = ctypes.c_void_p()
    # bucket_count < 1 is rejected before any device work (concurrent_hash.py:96-99)
    assert lib.vs_table_create(0, 4, 0, ctypes.byref(h)) == _lib.VS_ERR_INVALID
    with pytest.raises(ValueError):
        _lib.check(lib.vs_table_create(4, 0, 0, ctypes.byref(h)))
    assert "excess" in _lib.last_error()
    assert lib.vs_hash_keys(None, 0, 0, None, None) == _lib.VS_ERR_INVALID


def test_product_refuses_to_run_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: the refusal path is for CPU-only hosts")
    from paper_1805_03709_b200 import BlockHashSet, NativeUnavailable

    with pytest.raises(NativeUnavailable):
        BlockHashSet(64, 64)
    # argument validation still mirrors the reference before the device check
    with pytest.raises(ValueError):
        BlockHashSet(0, 64)
    with pytest.raises(ValueError):
        BlockHashSet(64, 64, lock_stripes=3)


def test_product_does_not_import_oracle():
    import pathlib

    pkg = pathlib.Path(_lib.__file__).parent
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
