"""Fused INT8 QKV GEMM + attention (csrc/qkv_attention.cuh) parity.

The engine runs the fused kernel for INT8-attention layers whenever every attention tile's
keys fit one 128-row tile (all sequences S <= 128; S in {32, 64} packed).  It must give the
same codes as the two-kernel path and the reference (encoder.py:355-379) bit for bit:
  * stage by stage (teacher-forced: q|k|v codes and ctx codes against the oracle);
  * end to end against the oracle (FULLY_QUANT, MHA_ONLY);
  * fused vs unfused (SAMP_NO_QA_FUSED=1) on the same batch, for batches whose work items
    (tiles x heads) wrap the persistent grid several times, with padding (att < S),
    packed S = 32 / 64 tiles next to single-sequence tiles, and batch 1.
"""

import numpy as np
import pytest

from oracle import samp_oracle as orc
from paper_2209_09130_b200.plan import PrecisionPlan
from paper_2209_09130_b200.quantization import CalibrationTable
from paper_2209_09130_b200.synthetic import build_archive, tiny_vocab
from paper_2209_09130_b200.tokenization import EncodedInput

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def base2():
    vocab = tiny_vocab(max_seq_len=512, extra_tokens=[f"w{i}" for i in range(1000 - 44)])
    arch = build_archive(num_layers=2, hidden=768, num_heads=12, intermediate=3072, max_position=512, seed=7,
                         weight_scale=0.02, vocab=vocab, task="classification")
    model = orc.Model.from_manifest(arch.manifest, arch.tensors)
    table = CalibrationTable(model_fingerprint=arch.fingerprint)
    rng = np.random.default_rng(4)
    for _ in range(2):
        ids = rng.integers(4, 1000, 96).tolist()
        taps = {}
        orc.run(model, ids, [0] * len(ids), len(ids), orc.plan_prefix("FP", 2, 0), taps=taps)
        for site, v in taps.items():
            table.observe(site, v)
    arch.calibration = table
    return arch, {s: e.amax for s, e in table.entries.items()}


def _batch(rng, specs, V=1000):
    encs = []
    for total, att in specs:
        ids = rng.integers(4, V, size=att).tolist() + [2] * (total - att)
        segs = [0] * (total // 2) + [1] * (total - total // 2)
        encs.append(EncodedInput(ids, segs, att))
    return encs


def _engine(arch):
    from paper_2209_09130_b200.engine import Engine
    return Engine(arch)


def _run(arch, encs, plan, monkeypatch, fused, env=()):
    if fused:
        monkeypatch.delenv("SAMP_NO_QA_FUSED", raising=False)
    else:
        monkeypatch.setenv("SAMP_NO_QA_FUSED", "1")
    for k in env:
        monkeypatch.setenv(k, "1")
    eng = _engine(arch)   # fresh engine: no captured graph of the other path
    out = eng.run_batch(encs, plan).hidden_states.copy()
    eng.run_batch(encs, plan)   # graph replay (the counters are reset inside the graph)
    again = eng.run_batch(encs, plan).hidden_states.copy()
    np.testing.assert_array_equal(out, again)
    for k in ("SAMP_NO_QA_FUSED",) + tuple(env):
        monkeypatch.delenv(k, raising=False)
    return out


MIXED = [(128, 128), (128, 90), (64, 64), (64, 64), (64, 40), (32, 32), (32, 32), (32, 32), (32, 17),
         (96, 96), (100, 71), (64, 64), (17, 17), (128, 1)]


def test_fused_teacher_forced_stages(base2):
    arch, amax = base2
    eng = _engine(arch)
    H = 768
    rng = np.random.default_rng(21)
    encs = _batch(rng, MIXED)
    seq_start, _, _, _ = eng.pack(encs)
    T = int(seq_start[-1])
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    eng.set_capture(True)
    res = eng.run_batch(encs, plan)
    eng.set_capture(False)
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    for i in range(2):
        in_q = eng.fetch_stage("in_q", i, np.int8, (T, H))
        qkv = eng.fetch_stage("qkv_q", i, np.int8, (T, 3 * H))
        ctx = eng.fetch_stage("ctx_q", i, np.int8, (T, H))
        s_in = model.scale(orc.input_site(i))
        for s, enc in enumerate(encs):
            r0, r1 = seq_start[s], seq_start[s + 1]
            _, _, (qc, kc, vc) = orc.qkv_int8(model, i, in_q[r0:r1], s_in)
            np.testing.assert_array_equal(qkv[r0:r1], np.concatenate([qc, kc, vc], axis=1), err_msg=f"qkv L{i} s{s}")
            at = orc.attention_int8(model, i, qkv[r0:r1, :H], qkv[r0:r1, H:2 * H], qkv[r0:r1, 2 * H:],
                                    enc.attention_length)
            np.testing.assert_array_equal(ctx[r0:r1], at["ctx_q"], err_msg=f"attention L{i} s{s}")
    for s, enc in enumerate(encs):
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        np.testing.assert_array_equal(res.sequence(s), want, err_msg=f"hidden s{s}")


@pytest.mark.parametrize("mode", ["FULLY_QUANT", "MHA_ONLY"])
def test_fused_matches_oracle_end_to_end(base2, mode):
    arch, amax = base2
    eng = _engine(arch)
    rng = np.random.default_rng(5)
    encs = _batch(rng, [(128, 128), (64, 64), (64, 50), (32, 32), (77, 77)])
    plan = PrecisionPlan.prefix(mode, 2, 2)
    res = eng.run_batch(encs, plan)
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    for s, enc in enumerate(encs):
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        if mode == "FULLY_QUANT":
            np.testing.assert_array_equal(res.sequence(s), want)
        else:   # FP16 FFN: tolerance (test_gpu_engine.py)
            got = res.sequence(s)
            rel = float(np.linalg.norm(got - want) / np.linalg.norm(want))
            assert rel < 2e-2, rel


@pytest.mark.parametrize("specs", [
    [(128, 128)] * 32,                                   # C2: 384 items, 2.6 per CTA
    [(128, 128)] * 70 + [(128, 100)] * 10,               # 960 items: 6-7 per CTA
    [(64, 64)] * 150 + [(32, 32)] * 9 + [(64, 33)],      # packed tiles only
    MIXED * 6,
    [(128, 128)],                                        # batch 1: 12 items
], ids=["c2", "many_items", "packed", "mixed", "batch1"])
def test_fused_equals_unfused(base2, monkeypatch, specs):
    arch, _ = base2
    encs = _batch(np.random.default_rng(len(specs)), specs)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    fused = _run(arch, encs, plan, monkeypatch, True)
    ref = _run(arch, encs, plan, monkeypatch, False)
    np.testing.assert_array_equal(fused, ref)


@pytest.mark.parametrize("specs", [
    [(128, 128)] * 32,
    MIXED * 6,                                           # row tiles straddling packed / ragged tiles
    [(100, 100)] * 40 + [(64, 64)] * 7,                  # no row tile aligned with a sequence
    [(128, 128)],
], ids=["c2", "mixed", "ragged", "batch1"])
def test_row_tile_flags_equal_grid_wait(base2, monkeypatch, specs):
    """The out-projection reading its ctx rows by the fused kernel's per-tile counters
    (SAMP_QA_FLAGS=1, opt-in) equals waiting for the whole fused grid (default), bit for bit."""
    arch, _ = base2
    encs = _batch(np.random.default_rng(3 + len(specs)), specs)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    flags = _run(arch, encs, plan, monkeypatch, True, env=("SAMP_QA_FLAGS",))
    grid = _run(arch, encs, plan, monkeypatch, True)
    np.testing.assert_array_equal(flags, grid)


def test_fused_bert_large_geometry(monkeypatch):
    """H = 1024, 16 heads (BERT-large widths; K = 8 k-blocks, 3H biases in smem), S <= 128."""
    vocab = tiny_vocab(max_seq_len=512, extra_tokens=[f"w{i}" for i in range(1000 - 44)])
    arch = build_archive(num_layers=2, hidden=1024, num_heads=16, intermediate=4096, max_position=512, seed=9,
                         weight_scale=0.02, vocab=vocab, task="classification")
    model = orc.Model.from_manifest(arch.manifest, arch.tensors)
    table = CalibrationTable(model_fingerprint=arch.fingerprint)
    rng = np.random.default_rng(8)
    ids = rng.integers(4, 1000, 100).tolist()
    taps = {}
    orc.run(model, ids, [0] * len(ids), len(ids), orc.plan_prefix("FP", 2, 0), taps=taps)
    for site, v in taps.items():
        table.observe(site, v)
    arch.calibration = table
    amax = {s: e.amax for s, e in table.entries.items()}
    encs = _batch(np.random.default_rng(12), [(128, 128), (128, 70), (64, 64), (64, 64), (96, 96)] * 3)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    fused = _run(arch, encs, plan, monkeypatch, True)
    ref = _run(arch, encs, plan, monkeypatch, False)
    np.testing.assert_array_equal(fused, ref)
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    seq_start = np.concatenate([[0], np.cumsum([len(e.token_ids) for e in encs])])
    for s in (0, 1, 4):
        e = encs[s]
        want = orc.run(model, e.token_ids, e.segment_ids, e.attention_length, plan.layer_precisions)
        np.testing.assert_array_equal(fused[seq_start[s]:seq_start[s + 1]], want)
