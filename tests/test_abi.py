"""The C-ABI library builds for sm_100a, loads, and exports every symbol that
include/hf.h declares (no compute calls: this container has no GPU)."""

import ctypes as ct
import os
import subprocess

import pytest

from paper_1904_13131_b200 import _lib


def test_header_declares_the_bound_symbols():
    decl = set(_lib.header_symbols())
    assert decl == set(_lib._SIGS), sorted(decl ^ set(_lib._SIGS))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    for name in _lib.header_symbols():
        assert hasattr(L, name), name
    assert L.hf_abi_version() == 1
    assert L.hf_max_degree(2) == 8 and L.hf_max_degree(3) == 4


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_errors_do_not_need_a_device():
    L = _lib.lib()
    rc = L.hf_space_create(4, 2, 3, None, None, None, None, None, None, None, None, None, None, None)
    assert rc == _lib.HF_ERR_ARG
    assert "null" in _lib.last_error()
    assert L.hf_tangent_apply(None, None, None, None) == _lib.HF_ERR_ARG


def test_product_path_fails_loudly_without_cuda(monkeypatch):
    import torch

    from paper_1904_13131_b200 import device

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        device.require_cuda()


def test_pool_info_without_a_device():
    L = _lib.lib()
    pooled, live = ct.c_longlong(-1), ct.c_longlong(-1)
    assert L.hf_pool_release() == 0
    assert L.hf_pool_info(ct.byref(pooled), ct.byref(live)) == 0
    assert pooled.value == 0 and live.value >= 0
