"""Converter interop: an HF BERT checkpoint converted by the reference's own converter
(tests/golden/make_converted.py -> tests/golden/converted_bert/, reference
pkg/converter/src/samp_convert/convert.py:180) loads through this package's archive reader
and runs on the B200 engine; logits are checked against the source framework's (torch)
logits in the reference's parity fixture (fixture.py:50), the acceptance check of
reference pkg/converter/tests/test_convert.py:176-193 (there: 1e-4 for its FP32 engine).

CPU: the oracle (the reference's FP32 arithmetic) on the converted archive is within 1e-4
of torch — pins the layout reading and the encode path.
GPU: the engine's FP plan (FP16 tensor cores) within 2e-3 abs of torch (FP16 tolerance);
FULLY_QUANT after on-device calibration bit-exact with the oracle under the same scales.
"""

import json
import os

import numpy as np
import pytest

from oracle import samp_oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))
CONVERTED = os.path.join(HERE, "golden", "converted_bert")


def _load():
    from paper_2209_09130_b200.archive import load_archive
    arch = load_archive(CONVERTED)
    with open(os.path.join(CONVERTED, "parity.json")) as fh:
        doc = json.load(fh)
    return arch, doc


def test_converted_archive_oracle_matches_torch():
    from paper_2209_09130_b200.tokenization import encode
    arch, doc = _load()
    m = arch.manifest
    assert m.hidden // m.num_heads == 64
    model = orc.Model.from_manifest(m, arch.tensors)
    for text, want in zip(doc["inputs"], doc["logits"]):
        enc = encode(arch.vocab, text)
        h = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, orc.plan_prefix("FP", m.num_layers, 0))
        lg, _, _ = orc.classify_logits(model, h)
        np.testing.assert_allclose(lg, want, atol=1e-4)


@pytest.mark.gpu
def test_converted_archive_on_engine():
    from paper_2209_09130_b200.engine import Engine
    from paper_2209_09130_b200.plan import PrecisionPlan
    from paper_2209_09130_b200.tasks import classify
    arch, doc = _load()
    L = arch.manifest.num_layers
    eng = Engine(arch)
    encs = [eng.encode_text(t) for t in doc["inputs"]]
    fp = PrecisionPlan.prefix("FP", L, 0)
    worst = 0.0
    for enc, want in zip(encs, doc["logits"]):
        res = classify(arch, eng.run(enc, fp))
        worst = max(worst, float(np.max(np.abs(np.asarray(res.logits) - np.asarray(want)))))
    print(f"converted BERT, FP16 engine vs torch: max |d logit| = {worst:.2e}")
    assert worst < 2e-3
    # INT8: calibrate on the device, then the fully-quantized chain is bit-exact with the
    # oracle under the same scales
    arch.calibration = eng.calibrate(encs)
    model = orc.Model.from_manifest(arch.manifest, arch.tensors,
                                    {s: e.amax for s, e in arch.calibration.entries.items()})
    q = PrecisionPlan.prefix("FULLY_QUANT", L, L)
    batch = eng.run_batch(encs, q)
    for s, enc in enumerate(encs):
        want = orc.run(model, enc.token_ids, enc.segment_ids, enc.attention_length, q.layer_precisions)
        np.testing.assert_array_equal(batch.sequence(s), want)
