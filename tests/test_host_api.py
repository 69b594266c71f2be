"""Host-side logic of the drop-in API (no GPU): plans, sites, archive format, synthetic
weights, tokenizer, calibration tables, trace-derived cost contracts, selection rules."""

import json
import os

import numpy as np
import pytest

from conftest import load_case
from paper_2209_09130_b200 import allocator as al
from paper_2209_09130_b200.archive import ModelManifest, load_archive, write_archive
from paper_2209_09130_b200.errors import (CalibrationError, ConfigurationError, DataFormatError,
                                          FormatError, InfeasibleError, LoadError)
from paper_2209_09130_b200.plan import (FFN_ONLY, FP, FULLY_QUANT, MHA_ONLY, PrecisionPlan,
                                        activation_sites)
from paper_2209_09130_b200.quantization import CalibrationTable, code_usage, quantize, requantize_i32
from paper_2209_09130_b200.synthetic import build_archive, tiny_vocab
from paper_2209_09130_b200.tokenization import SPECIAL_TOKENS, EncodedInput, Vocab, encode, tokenize, wordpiece
from paper_2209_09130_b200.trace import OpTrace, record_forward


# ---------------------------------------------------------------- plans (encoder.py:86-136)

def test_prefix_plans_and_modes():
    p = PrecisionPlan.prefix(FULLY_QUANT, 4, 2)
    assert p.layer_precisions == ("FULL_INT8", "FULL_INT8", "FP", "FP")
    assert p.quantized_layer_count == 2
    assert PrecisionPlan.prefix(FFN_ONLY, 3, 3).layer_precisions == ("FFN_ONLY_INT8",) * 3
    assert PrecisionPlan.prefix(MHA_ONLY, 2, 1).layer_precisions == ("MHA_ONLY_INT8", "FP")
    with pytest.raises(ConfigurationError):
        PrecisionPlan.prefix(FP, 3, 1)
    with pytest.raises(ConfigurationError):
        PrecisionPlan.prefix(FULLY_QUANT, 3, 4)
    with pytest.raises(ConfigurationError):
        PrecisionPlan(FFN_ONLY, ("FULL_INT8",))
    with pytest.raises(ConfigurationError):
        PrecisionPlan("NOPE", ("FP",))


def test_required_sites():
    full = PrecisionPlan.prefix(FULLY_QUANT, 2, 2).required_sites()
    assert full == set(activation_sites(2)) - {"L0.attn.in"}   # layer 0 input is embed.out
    ffn = PrecisionPlan.prefix(FFN_ONLY, 2, 1).required_sites()
    assert ffn == {"L0.ffn.in", "L0.ffn.mid"}
    mha = PrecisionPlan.prefix(MHA_ONLY, 2, 1).required_sites()
    assert mha == {"embed.out", "L0.attn.q", "L0.attn.k", "L0.attn.v", "L0.attn.softmax",
                   "L0.attn.out_in", "L0.ffn.in"}
    assert PrecisionPlan.prefix(FP, 2, 0).required_sites() == set()
    assert PrecisionPlan.prefix(FULLY_QUANT, 3, 2).codes() == bytes([2, 2, 0])


# ---------------------------------------------------------------- archive (archive.py)

def test_synthetic_generator_matches_reference_fingerprints():
    for case in ("tiny_cls", "mini", "base1"):
        meta, _ = load_case(case)
        recipe = dict(meta["recipe"])
        vocab = tiny_vocab(max_seq_len=recipe["max_position"],
                           extra_tokens=[f"w{i}" for i in range(meta["vocab_extra"])])
        assert build_archive(task=meta["task"], vocab=vocab, **recipe).fingerprint == meta["fingerprint"]
    # the reference's own checked-in calibration names this archive (tests/data/tiny_cls)
    assert build_archive(seed=0).fingerprint.startswith("7ede3e3d82fe8a98")


def test_archive_round_trip_and_errors(tmp_path):
    arch = build_archive(seed=4)
    arch.calibration = CalibrationTable(model_fingerprint=arch.fingerprint).set_amax("embed.out", 2.5)
    write_archive(arch, tmp_path / "a")
    back = load_archive(tmp_path / "a")
    assert back.fingerprint == arch.fingerprint
    for k, v in arch.tensors.items():
        np.testing.assert_array_equal(back.tensors[k], v)
    assert back.calibration.amax("embed.out") == 2.5
    with pytest.raises(ValueError):
        back.tensors["head.bias"][0] = 1.0              # frozen after load
    blob = (tmp_path / "a" / "tensors.bin").read_bytes()
    (tmp_path / "a" / "tensors.bin").write_bytes(blob[:-4])
    with pytest.raises(FormatError):
        load_archive(tmp_path / "a")
    with pytest.raises(LoadError):
        load_archive(tmp_path / "missing")
    with pytest.raises(LoadError):
        ModelManifest(1, 10, 3, 4, 5, 6, 2, 1e-12, "classification", 2)


# ---------------------------------------------------------------- quantization

def test_calibration_table_json_and_requirements():
    t = CalibrationTable(model_fingerprint="abc")
    t.observe("a", np.array([-3.0, 1.0])).observe("a", np.array([2.0]))
    assert t.amax("a") == 3.0
    back = CalibrationTable.from_json(t.to_json())
    assert back.model_fingerprint == "abc" and back.amax("a") == 3.0
    with pytest.raises(CalibrationError):
        t.require_all(["a", "b"])
    assert quantize(np.array([1.0, -0.5, 0.25], np.float32), 1 / 127).tolist() == [127, -64, 32]
    assert requantize_i32(np.array([100]), 0.5, 0.5, 1.0).tolist() == [25]
    rep = code_usage(np.array([-128, 0, 0, 127], np.int8))
    assert rep.used_count == 3 and rep.histogram[0] == 1


# ---------------------------------------------------------------- tokenizer

def _vocab(tokens, **kw):
    return Vocab.from_tokens(list(SPECIAL_TOKENS) + tokens, **kw)


def test_tokenizer_contracts():
    v = _vocab(["un", "##able", "##a", "##b", "##l", "##e", "to", "match", "hello", ",", "!", "cafe", "中", "文"])
    assert wordpiece(v, "unable") == ["un", "##able"]
    assert wordpiece(v, "xyz") == ["[UNK]"]
    assert tokenize(v, "HeLLo, Café!") == ["hello", ",", "cafe", "!"]
    assert tokenize(v, "中文") == ["中", "文"]
    assert wordpiece(v, "a" * 200) == ["[UNK]"]
    v8 = _vocab(["good", "bad"], max_seq_len=8)
    enc = encode(v8, "good", "bad bad")
    ids = v8.token_to_id
    assert enc.token_ids == [v8.cls_id, ids["good"], v8.sep_id, ids["bad"], ids["bad"], v8.sep_id,
                             v8.pad_id, v8.pad_id]
    assert enc.segment_ids == [0, 0, 0, 1, 1, 1, 1, 1] and enc.attention_length == 6
    v6 = _vocab(["a", "b"], max_seq_len=6)
    assert encode(v6, "a a a a a a", "b").token_ids == [v6.cls_id, 4, 4, v6.sep_id, 5, v6.sep_id]
    with pytest.raises(ConfigurationError):
        Vocab.from_tokens(["[CLS]", "[SEP]", "[PAD]", "a"])
    with pytest.raises(AttributeError):
        EncodedInput([1], [0], 1).attention_length = 2


# ---------------------------------------------------------------- trace-derived contracts

def test_trace_cost_contracts():
    # fully quantized: 6 INT8 GEMMs per layer; FFN-only: 2 INT8 + 4 F32 (reference
    # tests/test_acceptance.py:311-322); int8 boundaries between consecutive INT8 layers
    tr = OpTrace()
    record_forward(tr, PrecisionPlan.prefix(FULLY_QUANT, 3, 3).layer_precisions, 16, 64, 2, 128)
    assert tr.gemm_count("i8") == 18 and tr.gemm_count("f32") == 0
    assert [b.dtype for b in tr.boundaries] == ["f32", "i8", "i8", "i8", "i8", "f32"]
    tr = OpTrace()
    record_forward(tr, PrecisionPlan.prefix(FFN_ONLY, 3, 3).layer_precisions, 16, 64, 2, 128)
    assert tr.gemm_count("i8") == 6 and tr.gemm_count("f32") == 12
    assert tr.quant_count("quantize") == 6 and tr.quant_count("dequantize") == 0
    fp, q = OpTrace(), OpTrace()
    record_forward(fp, PrecisionPlan.prefix(FP, 2, 0).layer_precisions, 128, 768, 12, 3072)
    record_forward(q, PrecisionPlan.prefix(FULLY_QUANT, 2, 2).layer_precisions, 128, 768, 12, 3072)
    assert q.gemm_bytes() < fp.gemm_bytes() / 2


# ---------------------------------------------------------------- allocator (allocator.py)

def _profile(acc, lat, speed=None, mode=FULLY_QUANT):
    base = lat[0]
    speed = speed or [base / l for l in lat]
    return al.Profile(mode, [al.ProfilePoint(i, a, l, s) for i, (a, l, s) in enumerate(zip(acc, lat, speed))])


@pytest.mark.parametrize("acc,lat,sem,want", [
    ([0.9], [10.0], "latency", 0),
    ([0.90, 0.89, 0.80], [10.0, 8.0, 6.0], "latency", 1),        # dr 0.005 then 0.045
    ([0.5, 0.5, 0.5], [1.0, 2.0, 3.0], "latency", 1),            # dr 0 accepted once
    ([0.5, 0.6, 0.7], [3.0, 2.0, 1.0], "latency", 2),            # negative dr always accepted
    ([0.9, 0.8, 0.7], [1.0, 1.0, 0.5], "latency", 2),            # equal cost skipped
    ([0.9, 0.8, 0.7, 0.6], [4.0, 3.0, 2.0, 1.0], "speedup", 3),  # degenerates to the last point
    ([0.9, 0.8, 0.7, 0.6], [4.0, 3.0, 2.0, 1.0], "latency", 1),
])
def test_decay_aware_hand_traces(acc, lat, sem, want):
    # the same traces the reference's tests pin (reference tests/test_allocator.py:39-71)
    assert al.allocate_decay_aware(_profile(acc, lat), sem) == want


def test_selectors_and_ranking():
    assert al.select_by_latency_threshold(_profile([0.7, 0.9, 0.8], [3.0, 2.0, 1.0]), float("inf")) == 1
    assert al.select_by_accuracy_threshold(_profile([0.9, 0.7, 0.8], [3.0, 1.0, 2.0]), float("-inf")) == 1
    tie = _profile([0.9, 0.9, 0.9], [3.0, 2.0, 2.0])
    assert al.select_by_latency_threshold(tie, 10.0) == 0
    assert al.select_by_accuracy_threshold(tie, 0.5) == 1
    with pytest.raises(InfeasibleError, match="1"):
        al.select_by_latency_threshold(_profile([0.9, 0.8], [2.0, 1.0]), 0.5)
    with pytest.raises(InfeasibleError, match="0.6"):
        al.select_by_accuracy_threshold(_profile([0.6, 0.5], [2.0, 1.0]), 0.95)
    assert al.rank_by_ratio(_profile([0.80, 0.85, 0.70], [3.0, 2.0, 1.0]))[0] == 1
    spd = [1.0, 3.0, 2.0, 4.0]
    assert al.rank_by_ratio(_profile([0.9, 0.8, 0.8, 0.8], [1 / s for s in spd], spd)) == [3, 1, 2]
    assert al.rank_by_ratio(_profile([0.9], [1.0])) == []
    prof = _profile([0.90, 0.89, 0.80], [10.0, 8.0, 6.0])
    back = al.Profile.from_json(prof.to_json())
    assert back.points == prof.points and back.mode == prof.mode
    with pytest.raises(DataFormatError):
        al.Profile.from_json("{}")
    assert al.sweep_layer_counts(12, 5) == [0, 5, 10, 12]
    with pytest.raises(ConfigurationError):
        al.Profile(FULLY_QUANT, [al.ProfilePoint(2, 1, 1, 1), al.ProfilePoint(1, 1, 1, 1)])
    with pytest.raises(ConfigurationError):
        al.allocate_decay_aware(prof, "throughput")


def test_encoder_module_mirrors_reference_names():
    """`samp.encoder` users find the reference module's public names (encoder.py:45-87,
    :139-142, :421) in paper_2209_09130_b200.encoder."""
    from paper_2209_09130_b200 import encoder as enc
    for name in ("FP", "FULLY_QUANT", "FFN_ONLY", "LAYER_FP", "LAYER_FFN_INT8", "LAYER_FULL_INT8", "EMBED_OUT_SITE",
                 "ATTENTION_MASK_VALUE", "attn_in_site", "attn_site", "ffn_site", "activation_sites",
                 "PrecisionPlan"):
        assert hasattr(enc, name), name
    assert (enc.FP, enc.FULLY_QUANT, enc.FFN_ONLY) == ("FP", "FULLY_QUANT", "FFN_ONLY")
    assert (enc.LAYER_FFN_INT8, enc.LAYER_FULL_INT8, enc.EMBED_OUT_SITE) == ("FFN_ONLY_INT8", "FULL_INT8", "embed.out")
    sites = enc.activation_sites(2)
    assert sites[0] == "embed.out" and len(sites) == 1 + 8 * 2
    assert enc.ATTENTION_MASK_VALUE == np.float32(-10000.0)


def test_calibration_key_tracks_every_table_edit():
    """Engine._calibration_key (the per-forward check before the device amax push) must move on
    every edit the reference's fresh read would see, and stay put otherwise."""
    from paper_2209_09130_b200.engine import Engine
    from paper_2209_09130_b200.quantization import CalibrationTable, QuantScale

    class _E:
        pass

    table = CalibrationTable(model_fingerprint="x")
    for i, s in enumerate(("L0.attn.q", "L0.attn.k", "L0.ffn.mid")):
        table.set_amax(s, 1.0 + i)
    e = _E()
    e.archive = _E()
    e.archive.calibration = table
    key = lambda: Engine._calibration_key(e)   # noqa: E731
    k = key()
    assert key() == k
    edits = [
        lambda: setattr(table.entries["L0.ffn.mid"], "amax", 7.0),                       # in-place amax
        lambda: table.entries.__setitem__("L0.attn.q", QuantScale("L0.attn.q", 1.0)),    # replaced object
        lambda: table.entries.update({"L0.attn.q": table.entries["L0.attn.k"],
                                      "L0.attn.k": table.entries["L0.attn.q"]}),          # swapped objects
        lambda: table.entries.pop("L0.attn.k"),                                           # deleted
        lambda: setattr(table, "entries", dict(table.entries)),                           # dict replaced
    ]
    for edit in edits:
        edit()
        k2 = key()
        assert k2 != k
        k = k2
        assert key() == k
    e.archive.calibration = None
    assert key() is None
