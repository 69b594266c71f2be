"""Generate golden fixtures by running the REAL reference (build container only).

    python tests/golden/make_golden.py

Imports /root/reference/pkg/src/samp (staged with the restated tokenizer, see
refimport.py) and records, for a few deterministic synthetic models:
  * the archive recipe (build_archive kwargs) and its SHA-256 fingerprint, so
    tests can regenerate identical weights without storing them;
  * the reference calibration table (Engine.calibrate);
  * inputs, and for each precision plan the reference Engine.run hidden
    states, taps (capture_taps=True) and head outputs.
Outputs go to tests/golden/*.npz + *.json.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from refimport import load_reference  # noqa: E402

samp = load_reference()
from samp.encoder import Engine, PrecisionPlan  # noqa: E402
from samp.synthetic import build_archive, calibrated_archive, tiny_vocab  # noqa: E402
from samp.tasks import classify, tag  # noqa: E402
from samp.tokenization import EncodedInput  # noqa: E402


def random_inputs(vocab_size, specs, seed):
    """specs: list of (padded_len, att_len); ids past att_len are [PAD]=2."""
    rng = np.random.default_rng(seed)
    out = []
    for total, att in specs:
        ids = rng.integers(4, vocab_size, size=att).tolist() + [2] * (total - att)
        segs = [0] * total
        out.append(EncodedInput(ids, segs, att))
    return out


def dump_case(name, recipe, task, plans, inputs, calib_inputs=None, fp16_modes=(False,), taps_plan=None):
    vocab = recipe.pop("vocab_extra", None)
    kwargs = dict(recipe)
    if vocab is not None:
        kwargs["vocab"] = tiny_vocab(max_seq_len=kwargs["max_position"], extra_tokens=vocab)
    if calib_inputs is None:
        arch = calibrated_archive(task=task, **kwargs)
    else:
        arch = build_archive(task=task, **kwargs)
        arch.calibration = Engine(arch).calibrate(calib_inputs)
    arrays = {}
    meta = {
        "name": name,
        "recipe": {k: v for k, v in recipe.items()},
        "vocab_extra": len(vocab) if vocab is not None else 0,
        "task": task,
        "fingerprint": arch.fingerprint,
        "amax": {s: e.amax for s, e in arch.calibration.entries.items()},
        "inputs": [{"ids": e.token_ids, "segs": e.segment_ids, "att": e.attention_length} for e in inputs],
        "runs": [],
    }
    for fp16 in fp16_modes:
        eng = Engine(arch, fp16_storage=fp16)
        for mode, k in plans:
            plan = PrecisionPlan.prefix(mode, arch.manifest.num_layers, k)
            for j, enc in enumerate(inputs):
                want_taps = taps_plan == (mode, k) and not fp16 and j == 0
                out = eng.run(enc, plan, capture_taps=want_taps)
                key = f"{mode}.{k}.{int(fp16)}.{j}"
                arrays[f"hidden/{key}"] = out.hidden_states
                run = {"mode": mode, "k": k, "fp16": fp16, "input": j, "key": key}
                if task == "sequence_labeling":
                    res = tag(arch, out, enc.attention_length)
                else:
                    res = classify(arch, out)
                run["labels"] = res.label_ids
                arrays[f"logits/{key}"] = np.asarray(res.logits, dtype=np.float32)
                arrays[f"probs/{key}"] = np.asarray(res.scores, dtype=np.float32)
                if want_taps:
                    for site, val in out.taps.items():
                        arrays[f"taps/{key}/{site}"] = val
                    run["taps"] = sorted(out.taps)
                meta["runs"].append(run)
    # big arrays are pinned by SHA-256 of their float32 bytes (+ a head slice
    # for diagnostics) to keep the committed fixtures small
    small, digests = {}, {}
    for key, val in arrays.items():
        val = np.ascontiguousarray(val)
        if val.nbytes <= 64 * 1024:
            small[key] = val
        else:
            digests[key] = {"sha256": hashlib.sha256(val.tobytes()).hexdigest(),
                            "shape": list(val.shape), "dtype": str(val.dtype)}
            small[f"head/{key}"] = val.reshape(-1)[:512]
    meta["digests"] = digests
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **small)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(name, "runs", len(meta["runs"]), "arrays", len(arrays))


def main():
    # 1. the reference's own tiny_cls model (fingerprint 7ede3e3d...; reference tests/conftest.py:8-10)
    from samp.synthetic import SAMPLE_TEXTS
    arch_tmp = calibrated_archive(seed=0)
    eng = Engine(arch_tmp)
    tiny_inputs = [eng.encode_text(t) for t in SAMPLE_TEXTS[:4]]
    plans = [("FP", 0), ("FULLY_QUANT", 1), ("FULLY_QUANT", 2), ("FFN_ONLY", 1), ("FFN_ONLY", 2)]
    dump_case("tiny_cls", dict(seed=0, num_layers=2, hidden=8, num_heads=2, intermediate=16,
                               max_position=16), "classification", plans, tiny_inputs,
              fp16_modes=(False, True), taps_plan=("FULLY_QUANT", 2))

    # 2. mini model at GPU-legal shapes (head_dim 64), padded and unpadded inputs
    extra = [f"w{i}" for i in range(456)]   # vocab 500
    recipe = dict(seed=7, num_layers=2, hidden=128, num_heads=2, intermediate=256, max_position=64,
                  weight_scale=0.08, vocab_extra=extra)
    calib = random_inputs(500, [(64, 64), (64, 50), (64, 33), (64, 64)], seed=11)
    inputs = random_inputs(500, [(64, 64), (64, 40), (64, 17)], seed=12)
    plans = [("FP", 0), ("FULLY_QUANT", 1), ("FULLY_QUANT", 2), ("FFN_ONLY", 2)]
    # fp16 storage (reference --mode fp16, Engine(fp16_storage=True), encoder.py:428) too
    dump_case("mini", recipe, "classification", plans, inputs, calib_inputs=calib,
              fp16_modes=(False, True), taps_plan=("FULLY_QUANT", 2))

    # 3. one BERT-base-shaped layer (H=768, 12 heads, I=3072) at S=128: pins the
    #    768-wide LN tree and the 128-key softmax tree at the real sizes
    extra = [f"w{i}" for i in range(1000 - 44)]
    recipe = dict(seed=3, num_layers=1, hidden=768, num_heads=12, intermediate=3072, max_position=128,
                  weight_scale=0.02, vocab_extra=extra)
    calib = random_inputs(1000, [(128, 128), (128, 100)], seed=21)
    inputs = random_inputs(1000, [(128, 128), (128, 77)], seed=22)
    plans = [("FULLY_QUANT", 1), ("FFN_ONLY", 1), ("FP", 0)]
    dump_case("base1", recipe, "sequence_labeling", plans, inputs, calib_inputs=calib,
              fp16_modes=(False, True), taps_plan=("FULLY_QUANT", 1))


def analyze_golden():
    """The reference CLI's analyze-quant on its own tiny_cls model and infer inputs
    (reference tests/test_cli.py:255-263): CSV output + the token ids it ran on."""
    import contextlib
    import io
    from samp.cli import main as cli_main
    import tempfile
    from samp.archive import load_archive, write_archive
    data = "/root/reference/pkg/tests/data"
    # the snapshot's tests/data/tiny_cls lacks tensors.bin: rebuild the archive (same
    # fingerprint as its calibration.json) into a temp dir
    model_dir = os.path.join(tempfile.mkdtemp(prefix="samp_tiny_"), "tiny_cls")
    arch = calibrated_archive(seed=0)
    with open(f"{data}/tiny_cls/calibration.json") as fh:
        assert json.load(fh)["fingerprint"] == arch.fingerprint
    write_archive(arch, model_dir)
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli_main(["analyze-quant", "--model", model_dir, "--mode", "fully-quant",
                       "--format", "csv", "--data", f"{data}/infer_inputs.txt", "--sites", "L*.attn.softmax"])
    assert rc == 0
    eng = Engine(load_archive(model_dir))
    with open(f"{data}/infer_inputs.txt", encoding="utf-8") as fh:
        lines = [ln.rstrip("\n") for ln in fh if ln.strip()]
    encs = [eng.encode_text(ln) for ln in lines]
    doc = {"argv": "analyze-quant --mode fully-quant --format csv --sites L*.attn.softmax",
           "lines": lines,
           "inputs": [[list(map(int, e.token_ids)), list(map(int, e.segment_ids)), int(e.attention_length)]
                      for e in encs],
           "csv": buf.getvalue()}
    with open(os.path.join(HERE, "analyze_softmax.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    print("analyze_softmax.json", len(encs), "inputs")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()
elif __name__ == "__main__" and sys.argv[1] == "analyze":
    analyze_golden()


def bench_calibration(model="bert-base", n_seq=8, seq=128):
    """Reference Engine.calibrate for the bench model (SURVEY.md §8(d) recipe):
    BERT-shaped random init (seed 0, weight_scale 0.02, vocab 30522, max_position 512),
    8 default_rng(1) sequences of 128 ids, FP32 plan.  Written to bench_calibration_<model>.json."""
    from samp.synthetic import build_archive as ref_build
    shapes = {"bert-base": dict(num_layers=12, hidden=768, num_heads=12, intermediate=3072),
              "bert-large": dict(num_layers=24, hidden=1024, num_heads=16, intermediate=4096)}[model]
    vocab = tiny_vocab(max_seq_len=512, extra_tokens=[f"[unused{i}]" for i in range(30522 - 44)])
    arch = ref_build(task="classification", num_labels=2, max_position=512, seed=0, weight_scale=0.02,
                     vocab=vocab, **shapes)
    rng = np.random.default_rng(1)
    encs = [EncodedInput(rng.integers(0, 30522, size=seq).tolist(), [0] * seq, seq) for _ in range(n_seq)]
    table = Engine(arch).calibrate(encs)
    path = os.path.join(HERE, f"bench_calibration_{model}.json")
    with open(path, "w") as fh:
        fh.write(table.to_json() + "\n")
    print("wrote", path, len(table.entries), "sites")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--bench-calibration":
    bench_calibration(*(sys.argv[2:3] or ["bert-base"]))
