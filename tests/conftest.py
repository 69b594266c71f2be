import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_case(name):
    """Golden case written by tests/golden/make_golden.py from the real reference."""
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    return meta, arrays


def case_archive(meta):
    """Regenerate the case's archive with OUR synthetic generator (fingerprint-checked by tests)."""
    from paper_2209_09130_b200.quantization import CalibrationTable
    from paper_2209_09130_b200.synthetic import build_archive, tiny_vocab

    recipe = dict(meta["recipe"])
    recipe.pop("vocab_extra", None)
    extra = [f"w{i}" for i in range(meta["vocab_extra"])]
    vocab = tiny_vocab(max_seq_len=recipe["max_position"], extra_tokens=extra)
    arch = build_archive(task=meta["task"], vocab=vocab, **recipe)
    table = CalibrationTable(model_fingerprint=arch.fingerprint)
    for site, amax in meta["amax"].items():
        table.set_amax(site, amax)
    arch.calibration = table
    return arch


def golden_value(meta, arrays, key):
    """(array or None, sha256 or None) for a golden key."""
    if key in arrays:
        return arrays[key], None
    d = meta["digests"].get(key)
    return None, (d["sha256"] if d else None)


@pytest.fixture(scope="session")
def golden():
    return load_case
