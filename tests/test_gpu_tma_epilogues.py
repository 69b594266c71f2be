"""TMA-staged LayerNorm epilogues are bit-identical to the per-thread-store variants.

The LN GEMMs write their tiles through shared memory and TMA stores (int8 codes; small-batch
f32/f16 outputs in 128B/64B-swizzled boxes) and, at small batches, take the f32 residual
tile by TMA into the drained operand ring.  The arithmetic is unchanged, so every variant
(switches read per launch; a fresh engine per variant, no captured graph carried over; and
the 16-epilogue-warp LN variant, SAMP_LN_NE16)
must give the same hidden states bit for bit, for INT8 and FP16 plans, batch 1 (8-CTA
clusters) and batch 32 (4-CTA clusters), and a ragged final row tile.
"""

import numpy as np
import pytest

from oracle import samp_oracle as orc
from paper_2209_09130_b200.plan import PrecisionPlan
from paper_2209_09130_b200.quantization import CalibrationTable
from paper_2209_09130_b200.synthetic import build_archive, tiny_vocab
from paper_2209_09130_b200.tokenization import EncodedInput

pytestmark = pytest.mark.gpu

SWITCHES = ("SAMP_NO_LN_TMA_STORE", "SAMP_NO_LN_TMA_RES", "SAMP_LN96_STRIDED", "SAMP_LN_NE16")


@pytest.fixture(scope="module")
def arch2():
    vocab = tiny_vocab(max_seq_len=512, extra_tokens=[f"w{i}" for i in range(1000 - 44)])
    arch = build_archive(num_layers=2, hidden=768, num_heads=12, intermediate=3072, max_position=512, seed=11,
                         weight_scale=0.02, vocab=vocab, task="classification")
    model = orc.Model.from_manifest(arch.manifest, arch.tensors)
    table = CalibrationTable(model_fingerprint=arch.fingerprint)
    rng = np.random.default_rng(2)
    ids = rng.integers(4, 1000, 128).tolist()
    taps = {}
    orc.run(model, ids, [0] * len(ids), len(ids), orc.plan_prefix("FP", 2, 0), taps=taps)
    for site, v in taps.items():
        table.observe(site, v)
    arch.calibration = table
    return arch


def _run(arch, encs, plan, monkeypatch, env, fp16_storage=False):
    from paper_2209_09130_b200.engine import Engine
    for k in SWITCHES:
        monkeypatch.delenv(k, raising=False)
    for k in env:
        monkeypatch.setenv(k, "1")
    eng = Engine(arch, fp16_storage=fp16_storage)
    out = eng.run_batch(encs, plan).hidden_states.copy()
    for k in SWITCHES:
        monkeypatch.delenv(k, raising=False)
    return out


def _encs(n, S, seed):
    rng = np.random.default_rng(seed)
    return [EncodedInput(rng.integers(4, 1000, S).tolist(), [0] * S, S) for _ in range(n)]


@pytest.mark.parametrize("mode,k,fp16", [("FULLY_QUANT", 2, False), ("FP", 0, False), ("FP", 0, True),
                                         ("FFN_ONLY", 2, False)])
@pytest.mark.parametrize("batch", [1, 32, 5])
def test_tma_epilogue_variants_bit_identical(arch2, monkeypatch, mode, k, fp16, batch):
    encs = _encs(batch, 128 if batch != 5 else 100, batch)   # batch 5 x 100: a ragged last row tile
    plan = PrecisionPlan.prefix(mode, 2, k)
    base = _run(arch2, encs, plan, monkeypatch, (), fp16)
    for env in (("SAMP_NO_LN_TMA_STORE", "SAMP_NO_LN_TMA_RES"), ("SAMP_LN96_STRIDED",), ("SAMP_LN_NE16",)):
        other = _run(arch2, encs, plan, monkeypatch, env, fp16)
        np.testing.assert_array_equal(base, other, err_msg=f"{mode} batch {batch} {env}")


@pytest.mark.parametrize("mode,k,fp16", [("FULLY_QUANT", 2, False), ("FP", 0, True)])
@pytest.mark.parametrize("batch", [1, 5])
def test_ffn2_k_split_cluster(arch2, monkeypatch, mode, k, fp16, batch):
    """SAMP_LN_KS2: FFN2's two K halves on the two z-halves of a 16-CTA cluster, the partial
    accumulator tile pushed through DSMEM.  INT8: int32 adds, bit-identical; FP16: two f32
    partial sums (the tensor path's tolerance, test_gpu_engine.py)."""
    encs = _encs(batch, 128 if batch == 1 else 100, 7 + batch)
    plan = PrecisionPlan.prefix(mode, 2, k)
    base = _run(arch2, encs, plan, monkeypatch, (), fp16)
    monkeypatch.setenv("SAMP_LN_KS2", "1")
    from paper_2209_09130_b200.engine import Engine
    got = Engine(arch2, fp16_storage=fp16).run_batch(encs, plan).hidden_states.copy()
    monkeypatch.delenv("SAMP_LN_KS2")
    if mode == "FULLY_QUANT":
        np.testing.assert_array_equal(got, base)
    else:
        rel = float(np.linalg.norm(got - base) / np.linalg.norm(base))
        assert rel < 1e-3, rel


@pytest.mark.parametrize("batch", [1, 32, 5])
def test_gelu_fixup_path_bit_exact(arch2, monkeypatch, batch):
    """FFN1's fast GELU epilogue recomputes flagged 8-groups after its column loop
    (EpiGeluQuantT::gelu_fixup: TMEM re-read, exact numpy/SVML codes overwrite the fast ones).
    Flags are rare (~5e-4 of the groups), so SAMP_GELU_FIXUP_ALL sends EVERY group through
    the fixup: the codes must not change, and they equal the oracle's."""
    encs = _encs(batch, 128 if batch != 5 else 100, 40 + batch)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    base = _run(arch2, encs, plan, monkeypatch, ())
    monkeypatch.setenv("SAMP_GELU_FIXUP_ALL", "1")
    from paper_2209_09130_b200.engine import Engine
    got = Engine(arch2).run_batch(encs, plan).hidden_states.copy()
    monkeypatch.delenv("SAMP_GELU_FIXUP_ALL")
    np.testing.assert_array_equal(got, base)
    model = orc.Model.from_manifest(arch2.manifest, arch2.tensors,
                                    {s: e.amax for s, e in arch2.calibration.entries.items()})
    e = encs[0]
    want = orc.run(model, e.token_ids, e.segment_ids, e.attention_length, plan.layer_precisions)
    np.testing.assert_array_equal(got[:len(e.token_ids)], want)
