"""The CPU oracle against the real reference's golden vectors (no GPU).

Pins oracle/samp_oracle.py (+ oracle/npmath.c) bit-for-bit against fixtures
produced by running the reference itself (tests/golden/make_golden.py).
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import case_archive, golden_value, load_case
from oracle import samp_oracle as orc

F32 = np.float32


def _avx512_host():
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return all(f in flags for f in ("avx512f", "avx512bw", "avx512dq", "avx512vl", "avx512cd"))


@pytest.mark.skipif(not _avx512_host(), reason="numpy uses the SVML/AVX512 kernels only on AVX512 hosts")
@pytest.mark.parametrize("fn,ref", [("np_exp", np.exp), ("np_tanh", np.tanh)])
def test_npmath_matches_numpy(fn, ref):
    # exhaustive 2^32 sweeps were run when the restatement was written;
    # here: 4M random bit patterns + the ranges softmax / GELU actually use
    rng = np.random.default_rng(5)
    x = rng.integers(0, 2**32, size=1 << 22, dtype=np.uint64).astype(np.uint32).view(F32)
    x = np.concatenate([x, rng.uniform(-104, 0, 1 << 20).astype(F32), rng.uniform(-12, 12, 1 << 20).astype(F32)])
    with np.errstate(all="ignore"):
        want = ref(x)
    got = getattr(orc, fn)(x)
    same = (want.view(np.uint32) == got.view(np.uint32)) | (np.isnan(want) & np.isnan(got))
    assert same.all(), f"{np.count_nonzero(~same)} mismatches"


def test_pairwise_sum_restatement_matches_numpy():
    rng = np.random.default_rng(0)
    for n in list(range(1, 140)) + [191, 192, 250, 333, 384, 512, 768, 1024]:
        x = (rng.standard_normal(n) * 37).astype(F32)
        assert orc.pairwise_sum(x).view(np.int32) == np.sum(x).view(np.int32), n


def test_quantize_known_answers():
    # reference tests/test_quantization.py:25-35 KATs
    assert orc.quantize(np.array([1.0, -0.5, 0.25], F32), 1 / 127).tolist() == [127, -64, 32]
    assert orc.quantize(np.array([1e6, -1e6], F32), 0.01).tolist() == [127, -128]
    # half-away rounding on the F32 quotient, not round-half-even
    assert orc.quantize(np.array([0.5, -0.5, 1.5, 2.5], F32), 1.0).tolist() == [1, -1, 2, 3]


def test_gemm_i8_extremes():
    a = np.array([[127, -128]], np.int8)
    b = np.array([[1], [1]], np.int8)
    assert orc.gemm_i8(a, b).tolist() == [[-1]]


def _check(meta, arrays, key, got):
    want, digest = golden_value(meta, arrays, key)
    got = np.ascontiguousarray(np.asarray(got, dtype=F32))
    if want is not None:
        np.testing.assert_array_equal(got, want, err_msg=key)
    else:
        assert digest is not None, key
        assert hashlib.sha256(got.tobytes()).hexdigest() == digest, key


@pytest.mark.parametrize("case", ["tiny_cls", "mini", "base1"])
def test_oracle_reproduces_reference(case):
    meta, arrays = load_case(case)
    arch = case_archive(meta)
    assert arch.fingerprint == meta["fingerprint"], "synthetic generator diverged from the reference"
    L = arch.manifest.num_layers
    amax = {s: e.amax for s, e in arch.calibration.entries.items()}
    for fp16 in sorted({r["fp16"] for r in meta["runs"]}):
        model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax, fp16_storage=fp16)
        for run in (r for r in meta["runs"] if r["fp16"] == fp16):
            inp = meta["inputs"][run["input"]]
            taps = {} if "taps" in run else None
            hidden = orc.run(model, inp["ids"], inp["segs"], inp["att"],
                             orc.plan_prefix(run["mode"], L, run["k"]), taps=taps)
            _check(meta, arrays, f"hidden/{run['key']}", hidden)
            if meta["task"] == "sequence_labeling":
                logits, probs, labels = orc.tag_logits(model, hidden, inp["att"])
            else:
                logits, probs, label = orc.classify_logits(model, hidden)
                labels = [label]
            _check(meta, arrays, f"logits/{run['key']}", logits)
            _check(meta, arrays, f"probs/{run['key']}", probs)
            assert labels == run["labels"]
            if taps is not None:
                assert sorted(taps) == run["taps"]
                for site, val in taps.items():
                    _check(meta, arrays, f"taps/{run['key']}/{site}", val)
