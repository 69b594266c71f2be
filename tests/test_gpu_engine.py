"""End-to-end and teacher-forced parity of the B200 engine against the oracle.

INT8 path: bit-exact — every int8 code, every accumulator-derived value and the
final F32 hidden states equal the reference's (exp/tanh/pairwise restated).
FP16 path (FP layers, FFN-only MHA): tolerance, stated per test.
"""

import hashlib

import numpy as np
import pytest

from conftest import case_archive, golden_value, load_case
from oracle import samp_oracle as orc
from paper_2209_09130_b200.errors import CalibrationError, ConfigurationError, InputError
from paper_2209_09130_b200.plan import PrecisionPlan
from paper_2209_09130_b200.synthetic import build_archive, tiny_vocab
from paper_2209_09130_b200.quantization import CalibrationTable
from paper_2209_09130_b200.tokenization import EncodedInput

pytestmark = pytest.mark.gpu
F32 = np.float32

# FP16 tensor-core path vs the reference's FP32 math.  Hidden states are LayerNorm
# outputs (O(1)).  Plans that mix FP16 and INT8 can flip an INT8 code wherever the
# FP16 value sits near a rounding boundary, so the bound is relative-L2 plus a max.
FP16_REL_L2 = 2e-2
FP16_MAX_ABS = 0.3


def _fp16_close(got, want, label):
    rel = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))
    mx = float(np.max(np.abs(got - want)))
    print(f"{label}: rel_l2={rel:.2e} max_abs={mx:.2e}")
    assert rel < FP16_REL_L2 and mx < FP16_MAX_ABS, f"{label}: rel_l2 {rel:.3e} max {mx:.3e}"


def _engine(arch, fp16=False):
    from paper_2209_09130_b200.engine import Engine
    return Engine(arch, fp16_storage=fp16)


def _golden_equal(meta, arrays, key, got):
    want, digest = golden_value(meta, arrays, key)
    got = np.ascontiguousarray(got, dtype=F32)
    if want is not None:
        return np.array_equal(got, want), want
    return hashlib.sha256(got.tobytes()).hexdigest() == digest, None


@pytest.mark.parametrize("case", ["mini", "base1"])
def test_engine_matches_reference_goldens(case):
    meta, arrays = load_case(case)
    arch = case_archive(meta)
    L = arch.manifest.num_layers
    eng = _engine(arch)
    amax = {s: e.amax for s, e in arch.calibration.entries.items()}
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    for run in meta["runs"]:
        if run["fp16"]:
            continue
        inp = meta["inputs"][run["input"]]
        enc = EncodedInput(inp["ids"], inp["segs"], inp["att"])
        plan = PrecisionPlan.prefix(run["mode"], L, run["k"])
        out = eng.run(enc, plan)
        exact = run["mode"] == "FULLY_QUANT" and run["k"] == L
        ok, _ = _golden_equal(meta, arrays, f"hidden/{run['key']}", out.hidden_states)
        if exact:
            assert ok, f"{case} {run['key']}: INT8 path not bit-exact with the reference"
        else:
            want = orc.run(model, inp["ids"], inp["segs"], inp["att"], orc.plan_prefix(run["mode"], L, run["k"]))
            _fp16_close(out.hidden_states, want, f"{case} {run['key']}")


def _bert_like(num_layers=2, max_position=512, seed=5, task="classification"):
    vocab = tiny_vocab(max_seq_len=max_position, extra_tokens=[f"w{i}" for i in range(1000 - 44)])
    return build_archive(num_layers=num_layers, hidden=768, num_heads=12, intermediate=3072,
                         max_position=max_position, seed=seed, weight_scale=0.02, vocab=vocab, task=task)


def _calibrate_with_oracle(arch, seqs):
    model = orc.Model.from_manifest(arch.manifest, arch.tensors)
    table = CalibrationTable(model_fingerprint=arch.fingerprint)
    L = arch.manifest.num_layers
    for ids in seqs:
        taps = {}
        # FP forward (reference Engine.calibrate semantics) on the oracle
        orc.run(model, ids, [0] * len(ids), len(ids), orc.plan_prefix("FP", L, 0), taps=taps)
        for site, v in taps.items():
            table.observe(site, v)
    arch.calibration = table
    return {s: e.amax for s, e in table.entries.items()}


@pytest.fixture(scope="module")
def bert2():
    arch = _bert_like()
    rng = np.random.default_rng(3)
    amax = _calibrate_with_oracle(arch, [rng.integers(4, 1000, 64).tolist() for _ in range(2)])
    return arch, amax


def _batch(rng, specs, V=1000):
    encs = []
    for total, att in specs:
        ids = rng.integers(4, V, size=att).tolist() + [2] * (total - att)
        segs = [0] * (total // 2) + [1] * (total - total // 2)
        encs.append(EncodedInput(ids, segs, att))
    return encs


def test_stagewise_teacher_forced_int8(bert2):
    """Every fused kernel, fed the GPU's own stage inputs, equals the oracle stage bit-for-bit."""
    arch, amax = bert2
    eng = _engine(arch)
    L, H, I = 2, 768, 3072
    rng = np.random.default_rng(11)
    encs = _batch(rng, [(128, 128), (128, 77), (200, 200), (33, 33), (512, 300)])
    seq_start, att, ids, segs = eng.pack(encs)
    T = int(seq_start[-1])
    plan = PrecisionPlan.prefix("FULLY_QUANT", L, L)
    eng.set_capture(True)
    res = eng.run_batch(encs, plan)
    eng.set_capture(False)
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    st = {}
    for i in range(L):
        st[i] = {n: eng.fetch_stage(n, i, np.int8, (T, w)) for n, w in
                 (("in_q", H), ("qkv_q", 3 * H), ("ctx_q", H), ("ffn_in_q", H), ("mid_q", I))}
    for s, enc in enumerate(encs):
        r0, r1 = seq_start[s], seq_start[s + 1]
        # embed + quantize(embed.out)
        e = orc.embed(model, enc.token_ids, enc.segment_ids)
        np.testing.assert_array_equal(st[0]["in_q"][r0:r1], orc.quantize(e, model.scale("embed.out")))
        for i in range(L):
            g = {k: v[r0:r1] for k, v in st[i].items()}
            s_in = model.scale(orc.input_site(i))
            _, _, (qc, kc, vc) = orc.qkv_int8(model, i, g["in_q"], s_in)
            np.testing.assert_array_equal(g["qkv_q"], np.concatenate([qc, kc, vc], axis=1), err_msg=f"qkv L{i} s{s}")
            q, k, v = g["qkv_q"][:, :H], g["qkv_q"][:, H:2 * H], g["qkv_q"][:, 2 * H:]
            at = orc.attention_int8(model, i, q, k, v, enc.attention_length)
            np.testing.assert_array_equal(g["ctx_q"], at["ctx_q"], err_msg=f"attention L{i} s{s}")
            _, _, fin = orc.out_proj_int8(model, i, g["ctx_q"], g["in_q"], s_in)
            np.testing.assert_array_equal(g["ffn_in_q"], fin, err_msg=f"out-proj+LN L{i} s{s}")
            _, _, mid = orc.ffn1_int8(model, i, g["ffn_in_q"])
            np.testing.assert_array_equal(g["mid_q"], mid, err_msg=f"ffn1+gelu L{i} s{s}")
            site = f"L{i + 1}.attn.in" if i + 1 < L else None
            _, out_f, out_q = orc.ffn2_int8(model, i, g["mid_q"], g["ffn_in_q"], site)
            if site:
                np.testing.assert_array_equal(st[i + 1]["in_q"][r0:r1], out_q, err_msg=f"ffn2+LN L{i} s{s}")
            else:
                np.testing.assert_array_equal(res.hidden_states[r0:r1], out_f, err_msg=f"ffn2+LN L{i} s{s}")
        # and the whole forward
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        np.testing.assert_array_equal(res.sequence(s), want)


def test_batch_equals_single_runs(bert2):
    arch, _ = bert2
    eng = _engine(arch)
    rng = np.random.default_rng(2)
    encs = _batch(rng, [(64, 64), (130, 100), (17, 17)])
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    batch = eng.run_batch(encs, plan)
    for s, enc in enumerate(encs):
        np.testing.assert_array_equal(batch.sequence(s), eng.run(enc, plan).hidden_states)


@pytest.mark.parametrize("mode,k", [("FP", 0), ("FFN_ONLY", 2), ("FULLY_QUANT", 1), ("FFN_ONLY", 1)])
def test_fp16_and_mixed_plans_within_tolerance(bert2, mode, k):
    arch, amax = bert2
    eng = _engine(arch)
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    rng = np.random.default_rng(8)
    for enc in _batch(rng, [(64, 64), (96, 50)]):
        plan = PrecisionPlan.prefix(mode, 2, k)
        got = eng.run(enc, plan).hidden_states
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
        _fp16_close(got, want, f"{mode} k={k} S={len(enc.token_ids)}")


def test_classify_head_matches_oracle(bert2):
    from paper_2209_09130_b200.tasks import classify
    arch, amax = bert2
    eng = _engine(arch)
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    rng = np.random.default_rng(4)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    for enc in _batch(rng, [(64, 64), (40, 20)]):
        out = eng.run(enc, plan)
        res = classify(arch, out)
        lg, pr, lab = orc.classify_logits(model, out.hidden_states)
        np.testing.assert_allclose(res.logits, lg, rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(res.scores, pr, rtol=1e-5, atol=1e-6)
        if abs(pr[0] - pr[1]) > 1e-4:
            assert res.label_ids == [lab]


def test_errors_raised_before_compute(bert2):
    arch, _ = bert2
    eng = _engine(arch)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    with pytest.raises(InputError):
        eng.run(EncodedInput([0, 5000], [0, 0], 2), plan)
    with pytest.raises(InputError):
        eng.run(EncodedInput([], [], 0), plan)
    with pytest.raises(ConfigurationError):
        eng.run(EncodedInput([1, 2], [0, 0], 2), PrecisionPlan.prefix("FULLY_QUANT", 3, 1))
    saved = arch.calibration
    try:
        arch.calibration = CalibrationTable()
        with pytest.raises(CalibrationError):
            eng.run(EncodedInput([1, 2], [0, 0], 2), plan)
    finally:
        arch.calibration = saved


def test_gpu_calibration_matches_reference_semantics(bert2):
    """Engine.calibrate on the device (FP16 path + amax taps) vs the reference-style FP32
    calibration computed by the oracle on the same inputs."""
    arch, _ = bert2
    eng = _engine(arch)
    rng = np.random.default_rng(3)
    seqs = [rng.integers(4, 1000, 64).tolist() for _ in range(2)]     # the fixture's inputs
    table = eng.calibrate([EncodedInput(s, [0] * len(s), len(s)) for s in seqs])
    ref = _calibrate_with_oracle(_bert_like(), seqs)
    assert set(table.entries) == set(ref)
    worst = max(abs(table.amax(s) - a) / a for s, a in ref.items())
    print(f"max relative amax deviation {worst:.2e}")
    assert worst < 2e-2


def test_mha_only_extension_matches_composed_oracle(bert2):
    arch, amax = bert2
    eng = _engine(arch)
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    rng = np.random.default_rng(13)
    for enc in _batch(rng, [(64, 64), (80, 60)]):
        for k in (1, 2):
            plan = PrecisionPlan.prefix("MHA_ONLY", 2, k)
            got = eng.run(enc, plan).hidden_states
            want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)
            _fp16_close(got, want, f"MHA_ONLY k={k}")


def test_trace_and_sweep_on_device(bert2):
    from paper_2209_09130_b200 import allocator as al
    from paper_2209_09130_b200.trace import trace_ops
    arch, _ = bert2
    eng = _engine(arch)
    enc = EncodedInput(list(range(4, 68)), [0] * 64, 64)
    with trace_ops() as tr:
        eng.run(enc, PrecisionPlan.prefix("FULLY_QUANT", 2, 2))
    assert tr.gemm_count("i8") == 12 and tr.gemm_count("f32") == 0
    examples = [(" ".join(f"w{j}" for j in range(i, i + 20)), None, str(i % 2)) for i in range(6)]
    prof = al.build_profile(eng, "FULLY_QUANT", examples, layer_step=1, repeats=3, warmup=1)
    assert [p.quantized_layers for p in prof.points] == [0, 1, 2]
    assert prof.env["gemm_stats"]["2"]["int8_gemms"] == 12
    assert all(p.latency > 0 for p in prof.points)
    idx = al.allocate_decay_aware(prof)
    assert 0 <= idx < len(prof.points)


def test_cuda_graph_replay_is_bit_identical(bert2):
    arch, _ = bert2
    eng = _engine(arch)
    rng = np.random.default_rng(21)
    encs = _batch(rng, [(128, 128), (64, 40)])
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    outs = [eng.run_batch(encs, plan) for _ in range(4)]       # run, capture, replay, replay
    for o in outs[1:]:
        np.testing.assert_array_equal(o.hidden_states, outs[0].hidden_states)
        np.testing.assert_array_equal(o.logits, outs[0].logits)
    # geometry change invalidates nothing incorrectly
    other = eng.run_batch(encs[:1], plan)
    np.testing.assert_array_equal(other.sequence(0), outs[0].sequence(0))


def test_shared_engine_across_threads_is_bitwise_deterministic(bert2):
    """One Engine shared by several host threads (reference tests/test_encoder.py:340-350:
    results are bitwise thread-independent): concurrent run / run_batch calls with
    different plans and geometries equal the same calls made sequentially."""
    import threading
    arch, _ = bert2
    eng = _engine(arch)
    rng = np.random.default_rng(77)
    jobs = []
    for j in range(8):
        encs = _batch(rng, [(n, n) for n in rng.integers(16, 200, size=1 + j % 3).tolist()])
        encs = [EncodedInput(e.token_ids, e.segment_ids, len(e.token_ids) - j) for e in encs]
        mode = ("FULLY_QUANT", "FFN_ONLY", "FP", "MHA_ONLY")[j % 4]
        jobs.append((encs, PrecisionPlan.prefix(mode, 2, 0 if mode == "FP" else 2)))
    want = [eng.run_batch(encs, plan).hidden_states for encs, plan in jobs]
    got = [None] * len(jobs)

    def work(k):
        for _ in range(3):
            got[k] = eng.run_batch(*jobs[k]).hidden_states

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(jobs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for k in range(len(jobs)):
        np.testing.assert_array_equal(got[k], want[k], err_msg=f"job {k}")
