"""The drop-in boundary: libsamp_b200.so loads without a GPU and exports exactly the
C ABI declared in include/samp_b200.h; argument validation maps onto the reference's
exception classes before any device work."""

import ctypes
import os
import re

import pytest

from paper_2209_09130_b200 import _lib
from paper_2209_09130_b200.errors import ConfigurationError, DeviceError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "samp_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2209_09130_b200 import _build
        _build.build()
    return _lib.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(samp_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_the_header():
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_functions()) == bound


def test_device_check_fails_loudly_without_b200(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rc = lib.samp_device_check(0)
    assert rc == 5
    with pytest.raises(DeviceError):
        _lib.check(rc)


def test_create_validates_config_before_touching_the_device(lib):
    desc = _lib.ModelDesc(2, 96, 2, 128, 50, 16, 2, 2, 1e-12, 0)   # head_dim 48: unsupported
    h = ctypes.c_void_p()
    with pytest.raises(ConfigurationError):
        _lib.check(lib.samp_engine_create(ctypes.byref(desc), 0, ctypes.byref(h)))
    desc = _lib.ModelDesc(2, 128, 3, 128, 50, 16, 2, 2, 1e-12, 0)   # hidden % heads != 0
    with pytest.raises(ConfigurationError):
        _lib.check(lib.samp_engine_create(ctypes.byref(desc), 0, ctypes.byref(h)))


def test_engine_construction_without_gpu_raises_device_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2209_09130_b200.engine import Engine
    from paper_2209_09130_b200.synthetic import build_archive
    arch = build_archive(num_layers=1, hidden=128, num_heads=2, intermediate=256)
    with pytest.raises(DeviceError):
        Engine(arch)
