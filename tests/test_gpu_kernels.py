"""Kernel-level parity on the B200: raw tcgen05 GEMMs vs the oracle (exact for INT8)."""

import numpy as np
import pytest

from oracle import samp_oracle as orc
from paper_2209_09130_b200 import _lib

pytestmark = pytest.mark.gpu


def _gemm_i8(a, b):
    lib = _lib.load()
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), np.int32)
    _lib.check(lib.samp_debug_gemm_i8(_lib.ptr(np.ascontiguousarray(a)), _lib.ptr(np.ascontiguousarray(b)),
                                      _lib.ptr(c), m, n, k))
    return c


@pytest.mark.parametrize("m,n,k", [(128, 256, 128), (200, 96, 256), (4096, 2304, 768), (512, 768, 3072),
                                   (1, 64, 128), (333, 3072, 768)])
def test_gemm_i8_exact(m, n, k):
    rng = np.random.default_rng(m + n + k)
    a = rng.integers(-128, 128, size=(m, k), dtype=np.int8)
    b = rng.integers(-128, 128, size=(k, n), dtype=np.int8)
    np.testing.assert_array_equal(_gemm_i8(a, b), orc.gemm_i8(a, b))


def test_gemm_i8_extreme_codes():
    # reference tests/test_kernels.py:95-98 ([[127,-128]] . [[1],[1]] = -1), tiled up to legal shapes
    a = np.zeros((128, 128), np.int8)
    a[0, 0], a[0, 1] = 127, -128
    a[1, :] = -128
    b = np.zeros((128, 32), np.int8)
    b[0, 0] = b[1, 0] = 1
    b[:, 1] = -128
    c = _gemm_i8(a, b)
    np.testing.assert_array_equal(c, orc.gemm_i8(a, b))
    assert c[0, 0] == -1 and c[1, 1] == 128 * 128 * 128


@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (4096, 768, 768), (300, 3072, 768)])
def test_gemm_f16(m, n, k):
    rng = np.random.default_rng(7)
    a = rng.standard_normal((m, k)).astype(np.float16)
    b = (rng.standard_normal((k, n)) * 0.05).astype(np.float16)
    lib = _lib.load()
    c = np.empty((m, n), np.float32)
    _lib.check(lib.samp_debug_gemm_f16(_lib.ptr(a.view(np.uint16)), _lib.ptr(b.view(np.uint16)), _lib.ptr(c), m, n, k))
    want = a.astype(np.float64) @ b.astype(np.float64)
    np.testing.assert_allclose(c, want, rtol=1e-3, atol=1e-3)
