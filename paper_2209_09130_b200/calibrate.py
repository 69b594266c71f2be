"""On-device calibration: the reference's ``Engine.calibrate`` (encoder.py:446-454).

The reference runs an FP32 forward per input with ``capture_taps=True`` and min-max
observes every activation site (quantization.py:94-99).  Here all inputs run as one
packed FP plan forward on the GPU; the FP16 epilogues / attention / embedding fold
max|x| of every tapped tensor into a per-site device amax (one atomic per warp), so
no tap tensor is ever materialised.  The arithmetic is the FP16 tensor-core path, so
amax values agree with the reference's FP32 calibration to ~1e-3 relative
(tests/test_gpu_engine.py); use a reference-produced calibration.json when bit-exact
INT8 codes versus the reference are required.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .plan import activation_sites
from .quantization import CalibrationTable


def calibrate_engine(engine, encoded_inputs, max_tokens: int = 1 << 16) -> CalibrationTable:
    encs = list(encoded_inputs)
    table = CalibrationTable(model_fingerprint=engine.archive.fingerprint)
    sites = activation_sites(engine.manifest.num_layers)
    if not encs:
        return table
    for e in encs:
        engine._validate(e, engine.manifest)
    # chunk so one call's activations stay bounded
    chunk, tokens = [], 0
    batches = []
    for e in encs:
        if chunk and tokens + len(e.token_ids) > max_tokens:
            batches.append(chunk)
            chunk, tokens = [], 0
        chunk.append(e)
        tokens += len(e.token_ids)
    batches.append(chunk)
    out = (ctypes.c_double * len(sites))()
    for b in batches:
        seq_start, att, ids, segs = engine.pack(b)
        with engine._lock:     # the calibration forward reuses the engine's buffers
            _lib.check(engine._lib.samp_calibrate(engine.handle, len(b), seq_start.ctypes.data, att.ctypes.data,
                                                  ids.ctypes.data, segs.ctypes.data, out))
        for site, v in zip(sites, out):
            table.observe_amax(site, float(v))
    return table
