"""Engine state under changing batch shapes, calibration edits and concurrent callers.

Regressions for the round-1 review (ADVICE.md / VERDICT.md "weak" 3 and 9):
  * host staging buffers growing between a small and a large host-IO forward;
  * CUDA graphs captured before the per-batch geometry arrays were reallocated;
  * calibration edits made directly on ``table.entries`` (no API call) — the reference
    reads the table fresh on every run (encoder.py:456-470);
  * one Engine shared by threads while the calibration changes (reference
    tests/test_encoder.py:340-350: results bitwise thread-independent).
"""

import threading

import numpy as np
import pytest

from oracle import samp_oracle as orc
from paper_2209_09130_b200.plan import PrecisionPlan
from paper_2209_09130_b200.quantization import CalibrationTable, QuantScale
from paper_2209_09130_b200.synthetic import build_archive, tiny_vocab
from paper_2209_09130_b200.tokenization import EncodedInput

pytestmark = pytest.mark.gpu


def _arch():
    vocab = tiny_vocab(max_seq_len=512, extra_tokens=[f"w{i}" for i in range(1000 - 44)])
    arch = build_archive(num_layers=2, hidden=768, num_heads=12, intermediate=3072, max_position=512,
                         seed=5, weight_scale=0.02, vocab=vocab, task="classification")
    model = orc.Model.from_manifest(arch.manifest, arch.tensors)
    table = CalibrationTable(model_fingerprint=arch.fingerprint)
    rng = np.random.default_rng(3)
    for _ in range(2):
        ids = rng.integers(4, 1000, 64).tolist()
        taps = {}
        orc.run(model, ids, [0] * 64, 64, orc.plan_prefix("FP", 2, 0), taps=taps)
        for site, v in taps.items():
            table.observe(site, v)
    arch.calibration = table
    return arch


@pytest.fixture(scope="module")
def arch():
    return _arch()


def _engine(arch):
    from paper_2209_09130_b200.engine import Engine
    return Engine(arch)


def _oracle(arch, enc, plan):
    amax = {s: e.amax for s, e in arch.calibration.entries.items()}
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, amax)
    return orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, plan.layer_precisions)


def _seqs(rng, lens):
    return [EncodedInput(rng.integers(4, 1000, n).tolist(), [0] * n, n) for n in lens]


def test_small_large_small_host_forwards(arch):
    """run(1 seq) -> run_batch(>= 5000 tokens, staging buffers grow) -> run(1 seq): head
    outputs land in live buffers and every result equals the oracle."""
    eng = _engine(arch)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    rng = np.random.default_rng(1)
    one = _seqs(rng, [100])[0]
    first = eng.run(one, plan)
    np.testing.assert_array_equal(first.hidden_states, _oracle(arch, one, plan))
    big = _seqs(rng, [128] * 40)                       # 5120 tokens > the 8192/2 staging rows
    res = eng.run_batch(big, plan)
    for s in (0, 39):
        np.testing.assert_array_equal(res.sequence(s), _oracle(arch, big[s], plan))
    again = eng.run(one, plan)
    np.testing.assert_array_equal(again.hidden_states, first.hidden_states)
    np.testing.assert_array_equal(again.head["logits"], first.head["logits"])
    np.testing.assert_array_equal(again.head["labels"], first.head["labels"])


def test_graph_replay_after_geometry_arrays_grow(arch):
    """Capture a graph for a 2-sequence batch, run a batch of >64 sequences (the per-batch
    sequence / tile arrays are reallocated), then replay the first shape."""
    eng = _engine(arch)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    rng = np.random.default_rng(2)
    small = _seqs(rng, [64, 40])
    ref = [eng.run_batch(small, plan) for _ in range(3)]   # run, capture, replay
    many = _seqs(rng, [16 + (j % 5) for j in range(90)])   # 90 sequences, 90 tiles
    out_many = eng.run_batch(many, plan)
    np.testing.assert_array_equal(out_many.sequence(77), _oracle(arch, many[77], plan))
    for _ in range(2):                                     # replays of the first key
        got = eng.run_batch(small, plan)
        np.testing.assert_array_equal(got.hidden_states, ref[0].hidden_states)
        np.testing.assert_array_equal(got.logits, ref[0].logits)


def test_direct_table_edits_reach_the_device(arch):
    """Editing ``table.entries`` in place (no version bump) changes the next forward exactly
    as a fresh engine with the edited table computes it."""
    eng = _engine(arch)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    enc = _seqs(np.random.default_rng(4), [96])[0]
    saved = {s: e.amax for s, e in arch.calibration.entries.items()}
    try:
        base = eng.run(enc, plan).hidden_states
        eng.run(enc, plan)                                   # graph captured for this shape
        arch.calibration.entries["L0.ffn.mid"].amax *= 0.5   # mutate the QuantScale in place
        arch.calibration.entries["L1.attn.q"] = QuantScale("L1.attn.q", saved["L1.attn.q"] * 1.25)
        edited = eng.run(enc, plan).hidden_states
        assert not np.array_equal(edited, base)
        np.testing.assert_array_equal(edited, _oracle(arch, enc, plan))
        np.testing.assert_array_equal(edited, _engine(arch).run(enc, plan).hidden_states)
    finally:
        for s, a in saved.items():
            arch.calibration.entries[s] = QuantScale(s, a)
    np.testing.assert_array_equal(eng.run(enc, plan).hidden_states, base)


def test_calibration_swaps_while_threads_run_forwards(arch):
    """Threads run forwards while another swaps the archive's table between two
    calibrations: every result equals the one-table result for one of them (the plan
    check, the scale push and the forward are atomic per call)."""
    eng = _engine(arch)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 2, 2)
    rng = np.random.default_rng(6)
    encs = _seqs(rng, [128, 77, 33])
    t1 = arch.calibration
    t2 = CalibrationTable(model_fingerprint=arch.fingerprint)
    for s, e in t1.entries.items():
        t2.set_amax(s, e.amax * (0.8 if "ffn" in s else 1.1))
    want = {}
    for name, t in (("t1", t1), ("t2", t2)):
        arch.calibration = t
        want[name] = eng.run_batch(encs, plan).hidden_states
    assert not np.array_equal(want["t1"], want["t2"])
    stop = threading.Event()
    bad = []

    def swapper():
        k = 0
        while not stop.is_set():
            arch.calibration = (t1, t2)[k % 2]
            k += 1

    def worker():
        for _ in range(20):
            got = eng.run_batch(encs, plan).hidden_states
            if not (np.array_equal(got, want["t1"]) or np.array_equal(got, want["t2"])):
                bad.append(got)

    sw = threading.Thread(target=swapper)
    workers = [threading.Thread(target=worker) for _ in range(4)]
    sw.start()
    for w in workers:
        w.start()
    for w in workers:
        w.join()
    stop.set()
    sw.join()
    arch.calibration = t1
    assert not bad, f"{len(bad)} forwards mixed two calibrations"
