"""GELU fast-path fallback rate on the bench batch.  Needs a measurement build:
    python tools/build_variant.py flags SAMP_GELU_FLAG_COUNT=1
    SAMP_B200_LIB=abtest/flags/libsamp_b200.so python tools/gelu_flag_rate.py
"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
os.environ["SAMP_GELU_FLAGS"] = "1"
import numpy as np, bench
from paper_2209_09130_b200.engine import Engine
from paper_2209_09130_b200.plan import PrecisionPlan
arch = bench.build_model()
eng = Engine(arch)
plan = PrecisionPlan.prefix("FULLY_QUANT", 12, 12)
ss, att, ids, segs = bench.synthetic_batch(0)
eng._lib.samp_set_graphs(eng.handle, 0)
eng.forward_packed(plan, ss, att, ids, segs, hidden=False)
print("forward done")
