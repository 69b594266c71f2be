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


def _scales_from_bench():
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "bench_calibration_bert-base.json")
    amax = [v["amax"] for v in json.load(open(path))["sites"].values()]
    s = [float(np.float32(max(a, 127e-8) / 127.0)) for a in amax]
    rng = np.random.default_rng(0)
    s += list(np.float32(10.0 ** rng.uniform(-8, 2, 24)))
    s += [1.0, 0.5, 1 / 127, 2.0 ** -20, 3.0]
    return np.array(s, np.float32)


def test_quantize_fast_path_exhaustive():
    """quant_fast == quantize with the IEEE divide for every float x and 130 scales (all
    bench-calibration site scales + random ones): 5.6e11 comparisons on the device."""
    import ctypes
    lib = _lib.load()
    s = _scales_from_bench()
    bad = ctypes.c_ulonglong()
    _lib.check(lib.samp_debug_quant_exhaustive(_lib.ptr(s), len(s), ctypes.byref(bad)))
    assert bad.value == 0


def test_division_fast_path_exhaustive():
    import ctypes
    lib = _lib.load()
    d = np.concatenate([_scales_from_bench()[:40], np.array([1.0, 1.5, 7.0, 128.0, 511.9, 333.3], np.float32)])
    bad = ctypes.c_ulonglong()
    _lib.check(lib.samp_debug_div_exhaustive(_lib.ptr(d), len(d), ctypes.byref(bad)))
    assert bad.value == 0


def test_exp_fast_division_exhaustive():
    import ctypes
    lib = _lib.load()
    bad = ctypes.c_ulonglong()
    _lib.check(lib.samp_debug_exp_exhaustive(ctypes.byref(bad)))
    assert bad.value == 0


def test_exp2_fast_exhaustive():
    """Softmax fast exp (FFMA2 pairs, exact exponent add, unrefined reciprocal) equals numpy's
    float32 exp (IEEE divide restatement) for every float in [-86.5, 0]."""
    import ctypes
    lib = _lib.load()
    bad = (ctypes.c_ulonglong * 2)()
    _lib.check(lib.samp_debug_exp2_fast_exhaustive(bad))
    print(f"mismatches: unrefined {bad[0]}, refined {bad[1]}")
    assert bad[1] == 0
    assert bad[0] == 0


def test_gelu_fast_admission_all_bench_scales():
    """FFN1 fast GELU epilogue (MUFU gelu + margin flag, exact fallback): for every ffn.mid
    scale of the bench calibration plus extremes, no unflagged element over all floats
    |x| < 1e12 differs from quantize(gelu(x), s).  The engine runs this same check per scale
    before it may launch GELU_FAST (gelu_fast_prepare)."""
    import ctypes
    import json
    import os
    lib = _lib.load()
    path = os.path.join(os.path.dirname(__file__), "golden", "bench_calibration_bert-base.json")
    sites = json.load(open(path))["sites"]
    scales = [float(np.float32(max(v["amax"], 127e-8) / 127.0)) for k, v in sites.items() if k.endswith("ffn.mid")]
    scales += [float(np.float32(x)) for x in (1e-8, 1e-4, 0.01, 0.5, 3.0, 100.0)]
    counts = (ctypes.c_ulonglong * 2)()
    for s in scales:
        _lib.check(lib.samp_debug_gelu_fast_check(ctypes.c_float(s), counts))
        print(f"s={s:.4g}: mismatches {counts[0]}, flagged {counts[1]} ({counts[1] / 2**32:.2e})")
        assert counts[0] == 0


def test_gelu_finite_fast_path_exhaustive():
    import ctypes
    lib = _lib.load()
    bad = ctypes.c_ulonglong()
    _lib.check(lib.samp_debug_gelu_finite_exhaustive(ctypes.byref(bad)))
    assert bad.value == 0


@pytest.mark.parametrize("fn,name", [(0, "np_exp"), (1, "np_tanh")])
def test_device_transcendentals_equal_oracle(fn, name):
    lib = _lib.load()
    rng = np.random.default_rng(fn)
    x = np.concatenate([rng.integers(0, 2**32, 1 << 22, dtype=np.uint64).astype(np.uint32).view(np.float32),
                        rng.uniform(-104, 1, 1 << 21).astype(np.float32),
                        rng.uniform(-10, 10, 1 << 21).astype(np.float32)])
    y = np.empty_like(x)
    _lib.check(lib.samp_debug_unary(fn, _lib.ptr(x), _lib.ptr(y), x.size))
    want = getattr(orc, name)(x)
    same = (want.view(np.uint32) == y.view(np.uint32)) | (np.isnan(want) & np.isnan(y))
    assert same.all(), f"{np.count_nonzero(~same)} mismatches"


def test_device_gelu_equals_oracle():
    lib = _lib.load()
    x = np.random.default_rng(9).standard_normal(1 << 22).astype(np.float32) * 4
    y = np.empty_like(x)
    _lib.check(lib.samp_debug_unary(2, _lib.ptr(x), _lib.ptr(y), x.size))
    np.testing.assert_array_equal(y, orc.gelu(x))
