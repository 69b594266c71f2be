"""Parity at the geometries of BASELINE.json configs C3-C5.

The full configs (12/24 layers, thousands of sequences) are bench workloads; here each
geometry runs with 2 layers and a handful of sequences so the oracle finishes in
seconds, and the bar is the same as for BERT-base:
  * FULLY_QUANT k=L: every hidden state bit-exact with the oracle (reference
    encoder.py:333-418 restated in oracle/samp_oracle.py);
  * plans with FP16 layers: relative-L2 < 2e-2 and max-abs < 0.3 on the LayerNorm-scale
    hidden states (FP16 tensor cores vs the reference's FP32, see test_gpu_engine.py);
  * heads: logits within 1e-5 of the oracle (the reference's BLAS sgemm order is not
    replicable), argmax equal wherever the top-2 probabilities differ by > 1e-4.

C4: BERT-large geometry (H=1024, A=16, I=4096) NER `tag` head, S=256, FULLY_QUANT.
C5: text-matching sentence pairs (segment 1 after the first [SEP]), S=64, FFN_ONLY k=L,
    through run_batch and through the reference-shaped `tasks.match` API.
C3: the self-adaptive sweep grid k=0..L x {MHA_ONLY, FFN_ONLY, FULLY_QUANT} on one
    variable-length batch with S in [16, 512].
"""

import numpy as np
import pytest

from oracle import samp_oracle as orc
from paper_2209_09130_b200.plan import PrecisionPlan
from paper_2209_09130_b200.quantization import CalibrationTable
from paper_2209_09130_b200.synthetic import build_archive, tiny_vocab
from paper_2209_09130_b200.tokenization import EncodedInput

pytestmark = pytest.mark.gpu

FP16_REL_L2 = 2e-2
FP16_MAX_ABS = 0.3
LOGIT_TOL = 1e-5


def _fp16_close(got, want, label):
    rel = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))
    mx = float(np.max(np.abs(got - want)))
    print(f"{label}: rel_l2={rel:.2e} max_abs={mx:.2e}")
    assert rel < FP16_REL_L2 and mx < FP16_MAX_ABS, f"{label}: rel_l2 {rel:.3e} max {mx:.3e}"


def _archive(hidden, heads, inter, task, num_labels, seed, layers=2, max_position=512):
    vocab = tiny_vocab(max_seq_len=max_position, extra_tokens=[f"w{i}" for i in range(1000 - 44)])
    return build_archive(num_layers=layers, hidden=hidden, num_heads=heads, intermediate=inter,
                         max_position=max_position, seed=seed, weight_scale=0.02, vocab=vocab,
                         task=task, num_labels=num_labels)


def _calibrate(arch, seqs):
    """Reference Engine.calibrate semantics (FP forward, amax per site) on the oracle."""
    model = orc.Model.from_manifest(arch.manifest, arch.tensors)
    table = CalibrationTable(model_fingerprint=arch.fingerprint)
    L = arch.manifest.num_layers
    for ids, segs in seqs:
        taps = {}
        orc.run(model, ids, segs, len(ids), orc.plan_prefix("FP", L, 0), taps=taps)
        for site, v in taps.items():
            table.observe(site, v)
    arch.calibration = table
    return orc.Model.from_manifest(arch.manifest, arch.tensors,
                                   {s: e.amax for s, e in table.entries.items()})


def _engine(arch):
    from paper_2209_09130_b200.engine import Engine
    return Engine(arch)


# ---------------------------------------------------------------- C4: BERT-large NER
@pytest.fixture(scope="module")
def large_ner():
    arch = _archive(1024, 16, 4096, "sequence_labeling", 9, seed=7)
    rng = np.random.default_rng(17)
    model = _calibrate(arch, [(rng.integers(4, 1000, 96).tolist(), [0] * 96) for _ in range(2)])
    return arch, model


def test_c4_bert_large_geometry_int8_bit_exact_and_tag_head(large_ner):
    from paper_2209_09130_b200.tasks import tag
    arch, model = large_ner
    eng = _engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix("FULLY_QUANT", L, L)
    rng = np.random.default_rng(5)
    # two full S=256 rows, one padded row, one short row: packed in one call
    specs = [(256, 256), (256, 256), (256, 180), (40, 40)]
    encs = [EncodedInput(rng.integers(4, 1000, att).tolist() + [2] * (S - att), [0] * S, att) for S, att in specs]
    batch = eng.run_batch(encs, plan)
    for s, enc in enumerate(encs):
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        np.testing.assert_array_equal(batch.sequence(s), want, err_msg=f"BERT-large geometry seq {s}")
        # tag head through the reference-shaped API (per-token logits over the non-pad prefix)
        out = eng.run(enc, plan)
        np.testing.assert_array_equal(out.hidden_states, want)
        res = tag(arch, out, enc.attention_length)
        lg, pr, lab = orc.tag_logits(model, want, enc.attention_length)
        assert len(res.label_ids) == enc.attention_length
        np.testing.assert_allclose(np.asarray(res.logits), lg, rtol=LOGIT_TOL, atol=LOGIT_TOL)
        np.testing.assert_allclose(np.asarray(res.scores), pr, rtol=1e-5, atol=1e-6)
        top2 = np.sort(pr, axis=1)[:, -2:]
        decided = (top2[:, 1] - top2[:, 0]) > 1e-4
        assert np.array_equal(np.asarray(res.label_ids)[decided], np.asarray(lab)[decided])
    # batched device tag head (packed rows): the same per-token logits
    lg_all = np.concatenate([orc.tag_logits(model, batch.sequence(s), len(e.token_ids))[0]
                             for s, e in enumerate(encs)])
    np.testing.assert_allclose(batch.logits, lg_all, rtol=LOGIT_TOL, atol=LOGIT_TOL)


def test_c4_bert_large_geometry_mixed_plan(large_ner):
    arch, model = large_ner
    eng = _engine(arch)
    rng = np.random.default_rng(6)
    ids = rng.integers(4, 1000, 256).tolist()
    enc = EncodedInput(ids, [0] * 256, 256)
    for mode, k in (("FULLY_QUANT", 1), ("FP", 0)):
        plan = PrecisionPlan.prefix(mode, 2, k)
        got = eng.run(enc, plan).hidden_states
        want = orc.run(model, ids, enc.segment_ids, 256, plan.layer_precisions)
        _fp16_close(got, want, f"BERT-large {mode} k={k}")


# ---------------------------------------------------------------- C5: text matching
@pytest.fixture(scope="module")
def matcher():
    arch = _archive(768, 12, 3072, "text_matching", 2, seed=9, max_position=64)
    rng = np.random.default_rng(19)
    model = _calibrate(arch, [_pair(rng) for _ in range(2)])
    return arch, model


def _pair(rng, la=31, lb=30):
    """[CLS] a [SEP] b [SEP], segment 1 after the first [SEP] (SURVEY.md §8(d) C5 inputs)."""
    cls, sep = 0, 1
    ids = [cls] + rng.integers(4, 1000, la).tolist() + [sep] + rng.integers(4, 1000, lb).tolist() + [sep]
    segs = [0] * (la + 2) + [1] * (lb + 1)
    return ids, segs


def test_c5_text_matching_pairs_ffn_only(matcher):
    arch, model = matcher
    eng = _engine(arch)
    L = arch.manifest.num_layers
    assert eng.vocab.cls_id == 0 and eng.vocab.sep_id == 1
    rng = np.random.default_rng(23)
    pairs = [_pair(rng) for _ in range(48)]
    encs = [EncodedInput(ids, segs, len(ids)) for ids, segs in pairs]
    for mode in ("FFN_ONLY", "FULLY_QUANT"):
        plan = PrecisionPlan.prefix(mode, L, L)
        batch = eng.run_batch(encs, plan)
        assert batch.logits.shape == (len(encs), 2)
        agree = 0
        for s in range(0, len(encs), 6):       # oracle on a sample of the batch (FP32 GEMMs are slow)
            ids, segs = pairs[s]
            want = orc.run(model, ids, segs, len(ids), plan.layer_precisions)
            if mode == "FULLY_QUANT":
                np.testing.assert_array_equal(batch.sequence(s), want)
            else:
                _fp16_close(batch.sequence(s), want, f"pair {s} {mode}")
            # head on the device hidden states: the reference classify on those rows
            lg, pr, lab = orc.classify_logits(model, batch.sequence(s))
            np.testing.assert_allclose(batch.logits[s], lg, rtol=LOGIT_TOL, atol=LOGIT_TOL)
            agree += int(batch.labels[s] == lab or abs(pr[0] - pr[1]) <= 1e-4)
        assert agree == len(range(0, len(encs), 6))


def test_c5_match_api(matcher):
    from paper_2209_09130_b200.tasks import match
    arch, model = matcher
    eng = _engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix("FFN_ONLY", L, L)
    a = " ".join(f"w{i}" for i in range(3, 40))
    b = " ".join(f"w{i}" for i in range(50, 70))
    res = match(eng, plan, a, b)
    enc = eng.encode_text(a, b)
    assert 1 in enc.segment_ids and len(enc.token_ids) == 64
    out = eng.run(enc, plan)
    lg, pr, _ = orc.classify_logits(model, out.hidden_states)
    np.testing.assert_allclose(res.logits, lg, rtol=LOGIT_TOL, atol=LOGIT_TOL)
    np.testing.assert_allclose(res.scores, pr, rtol=1e-5, atol=1e-6)


# ---------------------------------------------------------------- C3: sweep grid
def test_c3_sweep_grid_varlen(request):
    arch = _archive(768, 12, 3072, "classification", 2, seed=5)
    rng = np.random.default_rng(3)
    model = _calibrate(arch, [(rng.integers(4, 1000, 64).tolist(), [0] * 64) for _ in range(2)])
    eng = _engine(arch)
    L = arch.manifest.num_layers
    rng = np.random.default_rng(0)
    lens = [16, 512] + rng.integers(16, 513, 4).tolist()       # S in [16, 512]
    encs = [EncodedInput(rng.integers(4, 1000, n).tolist(), [0] * n, n) for n in lens]
    seen = set()
    for mode in ("MHA_ONLY", "FFN_ONLY", "FULLY_QUANT"):
        for k in range(L + 1):
            plan = PrecisionPlan.prefix(mode, L, k)
            if plan.layer_precisions in seen:        # k = 0 is the all-FP plan in every mode
                continue
            seen.add(plan.layer_precisions)
            batch = eng.run_batch(encs, plan)
            for s in (0, 1, 2):
                enc = encs[s]
                want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
                if mode == "FULLY_QUANT" and k == L:
                    np.testing.assert_array_equal(batch.sequence(s), want, err_msg=f"S={lens[s]}")
                else:
                    _fp16_close(batch.sequence(s), want, f"{mode} k={k} S={lens[s]}")


# ---------------------------------------------------------------- packed attention tiles
def test_packed_short_sequences_bit_exact(matcher):
    """Runs of equal-length S=32 / S=64 sequences share one attention tile (block-diagonal
    packing, attention.cuh); mixed with unpackable lengths and padded rows (att < S)."""
    arch, model = matcher
    eng = _engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix("FULLY_QUANT", L, L)
    rng = np.random.default_rng(29)
    specs = [(64, 64), (64, 20), (32, 32), (32, 5), (32, 32), (32, 17), (32, 32), (40, 33),
             (64, 64), (64, 1), (64, 64), (16, 16), (32, 0), (32, 32)]
    encs = [EncodedInput(rng.integers(4, 1000, S).tolist(), [0] * (S // 2) + [1] * (S - S // 2), att)
            for S, att in specs]
    batch = eng.run_batch(encs, plan)
    for s, enc in enumerate(encs):
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        np.testing.assert_array_equal(batch.sequence(s), want, err_msg=f"seq {s} spec {specs[s]}")
    # same sequences one at a time (single-sequence tiles) give the same bits
    for s in (1, 3, 12):
        np.testing.assert_array_equal(eng.run(encs[s], plan).hidden_states, batch.sequence(s))


# ---------------------------------------------------------------- large token counts
@pytest.mark.parametrize("persistent", [False, True])
@pytest.mark.parametrize("geom", ["base", "large"])
def test_persistent_layernorm_gemms_bit_exact(geom, persistent, large_ner, monkeypatch):
    """T > 37 x 128 tokens: one-tile LN GEMMs over many waves, and (SAMP_LN_PERSISTENT=1) the
    persistent cluster GEMM (gemm_ln_persistent.cuh, st.async exchange of the LayerNorm
    partials): both bit-exact with the oracle."""
    if persistent:
        monkeypatch.setenv("SAMP_LN_PERSISTENT", "1")
    if geom == "large":
        arch, model = large_ner
        S, n = 256, 21                      # 5376 tokens
    else:
        arch = _archive(768, 12, 3072, "classification", 2, seed=5)
        rng = np.random.default_rng(3)
        model = _calibrate(arch, [(rng.integers(4, 1000, 64).tolist(), [0] * 64) for _ in range(2)])
        S, n = 128, 44                      # 5632 tokens
    eng = _engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix("FULLY_QUANT", L, L)
    rng = np.random.default_rng(31)
    encs = [EncodedInput(rng.integers(4, 1000, S).tolist(), [0] * S, S - (s % 3) * 7) for s in range(n)]
    batch = eng.run_batch(encs, plan)
    for s in (0, 1, n // 2, n - 1):
        enc = encs[s]
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        np.testing.assert_array_equal(batch.sequence(s), want, err_msg=f"{geom} seq {s}")


# ---------------------------------------------------------------- small batches: split-K
@pytest.mark.parametrize("lens", [[128], [100, 77], [40, 200, 60]])
def test_small_batch_splitk_layernorm_bit_exact(lens, monkeypatch):
    """T <= a few row tiles: out-projection / FFN2 run as split-K GEMMs into an int32
    workspace + the row LayerNorm kernel (ln_rows.cuh).  Bit-exact with the oracle and with
    the fused cluster kernel (default; the split-K path is opt-in, SAMP_SPLITK=1)."""
    monkeypatch.setenv("SAMP_SPLITK", "1")
    arch = _archive(768, 12, 3072, "classification", 2, seed=5)
    rng = np.random.default_rng(3)
    model = _calibrate(arch, [(rng.integers(4, 1000, 64).tolist(), [0] * 64) for _ in range(2)])
    eng = _engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix("FULLY_QUANT", L, L)
    rng = np.random.default_rng(41)
    encs = [EncodedInput(rng.integers(4, 1000, n).tolist(), [0] * n, n - 3) for n in lens]
    split = eng.run_batch(encs, plan)
    for s, enc in enumerate(encs):
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        np.testing.assert_array_equal(split.sequence(s), want, err_msg=f"seq {s}")
    monkeypatch.delenv("SAMP_SPLITK")
    eng2 = _engine(arch)
    fused = eng2.run_batch(encs, plan)
    np.testing.assert_array_equal(split.hidden_states, fused.hidden_states)
    # repeated calls (CUDA-graph replay) keep the workspace clean
    for _ in range(3):
        np.testing.assert_array_equal(eng.run_batch(encs, plan).hidden_states, split.hidden_states)


# ---------------------------------------------------------------- raw text in one call
def test_run_texts_equals_encoded_runs(matcher):
    """Engine.run_texts (native tokenizer + packed forward) == per-text encode_text + run."""
    arch, _ = matcher
    eng = _engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix("FFN_ONLY", L, L)
    words = ["w%d" % i for i in range(4, 300)]
    rng = np.random.default_rng(5)
    a = [" ".join(rng.choice(words, size=int(rng.integers(3, 40)))) for _ in range(12)]
    b = [" ".join(rng.choice(words, size=int(rng.integers(3, 40)))) for _ in range(12)]
    res = eng.run_texts(plan, a, b, hidden=True)
    for i in range(len(a)):
        enc = eng.encode_text(a[i], b[i])
        one = eng.run(enc, plan)
        np.testing.assert_array_equal(res.sequence(i), one.hidden_states)
        np.testing.assert_array_equal(res.logits[i], one.head["logits"][0])


@pytest.mark.parametrize("mode,k", [("FP", 0), ("FFN_ONLY", 2), ("MHA_ONLY", 2), ("FULLY_QUANT", 2)])
def test_persistent_layernorm_all_precisions_identical(mode, k, monkeypatch):
    """The persistent cluster LN GEMM (forced) gives bit-identical hidden states to the
    one-tile kernel for every layer kind: int8 and f16 accumulators, int8 / f32 residuals,
    quantized, dequantized (MHA-only) and f32/f16 outputs."""
    arch = _archive(768, 12, 3072, "classification", 2, seed=5)
    rng = np.random.default_rng(3)
    _calibrate(arch, [(rng.integers(4, 1000, 64).tolist(), [0] * 64) for _ in range(2)])
    plan = PrecisionPlan.prefix(mode, 2, k)
    rng = np.random.default_rng(43)
    encs = [EncodedInput(rng.integers(4, 1000, n).tolist(), [0] * n, n - 5) for n in (128, 96, 200, 64, 128)]
    base = _engine(arch).run_batch(encs, plan)
    monkeypatch.setenv("SAMP_LN_PERSISTENT", "1")
    pers = _engine(arch).run_batch(encs, plan)
    np.testing.assert_array_equal(pers.hidden_states, base.hidden_states)
    np.testing.assert_array_equal(pers.logits, base.logits)


def test_tiny_and_odd_sequence_lengths_bit_exact():
    """Sequences of 1..17 tokens (numpy pairwise leaves with n < 8, tails of 1..7, one-key
    softmax rows, single-row tiles) and att_len 0 / 1 / S, mixed in one packed batch."""
    arch = _archive(768, 12, 3072, "classification", 2, seed=5)
    rng = np.random.default_rng(3)
    model = _calibrate(arch, [(rng.integers(4, 1000, 64).tolist(), [0] * 64) for _ in range(2)])
    eng = _engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix("FULLY_QUANT", L, L)
    rng = np.random.default_rng(51)
    specs = [(1, 1), (2, 2), (7, 7), (8, 8), (9, 9), (15, 15), (16, 16), (17, 17), (2, 1), (9, 0), (13, 6), (1, 0)]
    encs = [EncodedInput(rng.integers(4, 1000, S).tolist(), [0] * S, att) for S, att in specs]
    batch = eng.run_batch(encs, plan)
    for s, enc in enumerate(encs):
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        np.testing.assert_array_equal(batch.sequence(s), want, err_msg=f"spec {specs[s]}")


# ---------------------------------------------------------------- analyze-quant code usage
@pytest.mark.parametrize("mode,k", [("FULLY_QUANT", 2), ("FFN_ONLY", 2), ("FULLY_QUANT", 1)])
def test_code_usage_histograms_equal_oracle(matcher, mode, k):
    """Engine.code_usage (device histogram taps on the codes the kernels write) equals the
    reference's analyze-quant loop (cli.py:284-292: tap -> quantize -> code_usage, summed
    over inputs) on the oracle, for every site the plan quantizes; packed, padded rows."""
    from paper_2209_09130_b200.quantization import code_usage
    arch, model = matcher
    eng = _engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix(mode, L, k)
    rng = np.random.default_rng(31)
    specs = [(64, 64), (64, 20), (32, 32), (32, 5), (40, 33), (16, 16)]
    encs = [EncodedInput(rng.integers(4, 1000, S).tolist(), [0] * (S // 2) + [1] * (S - S // 2), att)
            for S, att in specs]
    got = eng.code_usage(encs, plan)
    assert set(got) == plan.required_sites()
    want = {}
    for enc in encs:
        taps = {}
        orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions, taps=taps)
        for site in got:
            r = code_usage(orc.quantize(taps[site], model.scale(site)), site)
            want[site] = want[site].merged(r) if site in want else r
    for site in sorted(got):
        if mode == "FULLY_QUANT":   # INT8 chain from the embedding: bit-exact codes
            assert got[site].histogram == want[site].histogram, site
        else:   # codes downstream of the FP16 tensor-core MHA: rounding flips only
            g, w = np.array(got[site].histogram), np.array(want[site].histogram)
            assert g.sum() == w.sum(), site
            assert np.abs(g - w).sum() <= 0.01 * w.sum(), (site, np.abs(g - w).sum(), w.sum())
    sm = [s for s in got if s.endswith("softmax")]
    if sm:   # heads x S x S probabilities per sequence, masked keys included
        heads = arch.manifest.num_heads
        assert sum(got[sm[0]].histogram) == heads * sum(S * S for S, _ in specs)
    # the reference-shaped analyze-quant entry point: fnmatch filter, sorted sites
    rep = eng.analyze_quant(encs, plan, "L0.ffn.*")
    assert list(rep) == sorted(s for s in plan.required_sites() if s.startswith("L0.ffn."))
    assert all(rep[s].histogram == got[s].histogram for s in rep)
    from paper_2209_09130_b200.errors import ConfigurationError, InputError
    with pytest.raises(InputError, match="matches nothing"):
        eng.analyze_quant(encs, plan, "nope*")
    with pytest.raises(ConfigurationError):
        eng.analyze_quant(encs, PrecisionPlan.prefix(mode, L, 0))
