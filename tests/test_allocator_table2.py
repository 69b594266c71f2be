"""Allocator fidelity on the paper's six published sweep profiles (SAMP Table 2: AFQMC,
IFLYTEK, TNEWS x {fully-quant, FFN-only}), the reference's acceptance criterion 1
(reference pkg/tests/test_acceptance.py:67-178).

Each sweep is (accuracy, speedup) at 0, 2, ..., 12 quantized layers.  Expected picks are
checked two ways: against an independent transcription of the allocation rules written
here (so a drifting implementation AND a drifting fixture are both caught), and against
the allocator of this package (paper_2209_09130_b200/allocator.py, restating reference
allocator.py:107-262).
"""

import pytest

from paper_2209_09130_b200.allocator import (InfeasibleError, Profile, ProfilePoint, allocate_decay_aware,
                                             rank_by_ratio, select_by_accuracy_threshold,
                                             select_by_latency_threshold)
from paper_2209_09130_b200.plan import FFN_ONLY, FULLY_QUANT

# SAMP Table 2 sweeps: accuracy and speedup per quantized-layer count {0, 2, ..., 12}
SWEEPS = {
    ("AFQMC", FULLY_QUANT): ([0.7338, 0.6671, 0.3167, 0.3188, 0.6435, 0.6874, 0.4409],
                             [3.3741, 3.5790, 3.7689, 4.0486, 4.3882, 4.7751, 5.1817]),
    ("IFLYTEK", FULLY_QUANT): ([0.6056, 0.5572, 0.2957, 0.1454, 0.1493, 0.1149, 0.0150],
                               [1.4870, 1.5550, 1.6144, 1.7305, 1.8645, 2.0162, 2.1978]),
    ("TNEWS", FULLY_QUANT): ([0.5632, 0.0930, 0.0856, 0.0952, 0.0851, 0.0900, 0.0884],
                             [3.5022, 3.6790, 3.9083, 4.2274, 4.5985, 4.9869, 5.3271]),
    ("AFQMC", FFN_ONLY): ([0.7338, 0.7340, 0.7318, 0.7088, 0.6872, 0.5588, 0.5279],
                          [3.3741, 3.4799, 3.6162, 3.7725, 4.0059, 4.2262, 4.4574]),
    ("IFLYTEK", FFN_ONLY): ([0.6056, 0.6007, 0.5932, 0.5840, 0.5786, 0.5663, 0.5641],
                            [1.4870, 1.5073, 1.5532, 1.6269, 1.7095, 1.7863, 1.8821]),
    ("TNEWS", FFN_ONLY): ([0.5632, 0.5654, 0.5640, 0.5610, 0.5523, 0.5208, 0.5077],
                          [3.5022, 3.6659, 3.7465, 3.9527, 4.1440, 4.3917, 4.6195]),
}

# point indices the rules pick (index i = 2i quantized layers)
EXPECTED = {
    ("AFQMC", FULLY_QUANT): dict(decay_latency=5, decay_speedup=2, top5=[5, 4, 6, 1, 3], min_acc=(0.60, 5)),
    ("IFLYTEK", FULLY_QUANT): dict(decay_latency=1, decay_speedup=6, top5=[1, 6, 5, 4, 3], min_acc=(0.40, 1)),
    ("TNEWS", FULLY_QUANT): dict(decay_latency=3, decay_speedup=4, top5=[6, 5, 4, 3, 2], min_acc=(0.09, 3)),
    ("AFQMC", FFN_ONLY): dict(decay_latency=1, decay_speedup=6, top5=[1, 2, 3, 4, 6], min_acc=(0.70, 3)),
    ("IFLYTEK", FFN_ONLY): dict(decay_latency=4, decay_speedup=6, top5=[6, 4, 5, 3, 2], min_acc=(0.5813, 3)),
    ("TNEWS", FFN_ONLY): dict(decay_latency=1, decay_speedup=6, top5=[2, 1, 3, 4, 5], min_acc=(0.5567, 3)),
}
# latency budget halfway between the 6- and 8-layer points
EXPECTED_LATENCY_PICK = {
    ("AFQMC", FULLY_QUANT): 5, ("IFLYTEK", FULLY_QUANT): 4, ("TNEWS", FULLY_QUANT): 5,
    ("AFQMC", FFN_ONLY): 4, ("IFLYTEK", FFN_ONLY): 4, ("TNEWS", FFN_ONLY): 4,
}


def _profile(key) -> Profile:
    acc, spd = SWEEPS[key]
    return Profile(mode=key[1], points=[ProfilePoint(2 * i, acc[i], 1.0 / spd[i], spd[i]) for i in range(len(acc))])


# ---- independent transcriptions of the rules (paper Algorithm 1 + Appendix A)
def _decay(acc, cost):
    best, rec_a, rec_c, pick = float("inf"), acc[0], cost[0], 0
    for i in range(1, len(acc)):
        if cost[i] == rec_c:
            continue
        rate = (acc[i] - rec_a) / (cost[i] - rec_c)
        if rate < 0 or rate < best:
            best, rec_a, rec_c, pick = rate, acc[i], cost[i], i
    return pick


def _ratio_rank(acc, spd, n=5):
    free = sorted((i for i in range(1, len(acc)) if acc[0] - acc[i] <= 0), key=lambda i: (-spd[i], i))
    paid = sorted((i for i in range(1, len(acc)) if acc[0] - acc[i] > 0),
                  key=lambda i: (-(spd[i] - spd[0]) / (acc[0] - acc[i]), i))
    return (free + paid)[:n]


@pytest.mark.parametrize("key", sorted(EXPECTED))
def test_allocator_on_published_sweep(key):
    acc, spd = SWEEPS[key]
    lat = [1.0 / s for s in spd]
    exp = EXPECTED[key]
    prof = _profile(key)
    assert _decay(acc, lat) == exp["decay_latency"] == allocate_decay_aware(prof, "latency")
    assert _decay(acc, spd) == exp["decay_speedup"] == allocate_decay_aware(prof, "speedup")
    assert _ratio_rank(acc, spd) == exp["top5"] == rank_by_ratio(prof, 5)
    thr, pick = exp["min_acc"]
    assert min((i for i in range(len(acc)) if acc[i] > thr), key=lambda i: (lat[i], i)) == pick
    assert select_by_accuracy_threshold(prof, thr) == pick
    budget = (lat[3] + lat[4]) / 2.0
    want = max((i for i in range(len(acc)) if lat[i] < budget), key=lambda i: (acc[i], -i))
    assert want == EXPECTED_LATENCY_PICK[key] == select_by_latency_threshold(prof, budget)


def test_headline_afqmc_ffn_only():
    """The paper's worked example: AFQMC FFN-only picks 2 layers by decay, 6 for accuracy
    >= 0.70, and ranks {2, 4, 6, 8, 12} layers as the top five."""
    prof = _profile(("AFQMC", FFN_ONLY))
    assert prof.points[allocate_decay_aware(prof)].quantized_layers == 2
    assert prof.points[select_by_accuracy_threshold(prof, 0.70)].quantized_layers == 6
    assert [prof.points[i].quantized_layers for i in rank_by_ratio(prof)] == [2, 4, 6, 8, 12]


def test_infeasible_thresholds_raise():
    prof = _profile(("TNEWS", FULLY_QUANT))
    with pytest.raises(InfeasibleError):
        select_by_accuracy_threshold(prof, 0.99)
    with pytest.raises(InfeasibleError):
        select_by_latency_threshold(prof, 1e-6)
