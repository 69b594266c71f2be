"""Per-kernel device times (CUDA events on the launching stream) for the bench model.

    python tools/profile_kernels.py [--batch 32] [--seq 128] [--plans FULLY_QUANT:12,FFN_ONLY:12,FP:0]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--seq", type=int, default=128)
    ap.add_argument("--plans", default="FULLY_QUANT:12,FFN_ONLY:12,FP:0")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import bench
    from paper_2209_09130_b200 import _lib
    from paper_2209_09130_b200.engine import Engine
    from paper_2209_09130_b200.plan import PrecisionPlan

    arch = bench.build_model()
    eng = Engine(arch)
    lib = _lib.load()
    seq_start, att, ids, segs = bench.synthetic_batch(0, args.batch, args.seq)
    for spec in args.plans.split(","):
        mode, k = spec.split(":")
        plan = PrecisionPlan.prefix(mode, 12, int(k))
        for _ in range(3):
            eng.forward_packed(plan, seq_start, att, ids, segs, hidden=False)
        _lib.check(lib.samp_set_profiling(eng.handle, 1))
        for _ in range(args.iters):
            eng.forward_packed(plan, seq_start, att, ids, segs, hidden=False)
        buf = ctypes.create_string_buffer(1 << 16)
        _lib.check(lib.samp_profile_report(eng.handle, buf, len(buf)))
        _lib.check(lib.samp_set_profiling(eng.handle, 0))
        prof = json.loads(buf.value.decode())
        tot = sum(v[0] for v in prof.values()) / args.iters
        print(f"== {mode} k={k} batch {args.batch} x {args.seq}: {tot * 1e3:.1f} us of kernels per forward")
        for name, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
            print(f"   {name:14s} {ms * 1e3 / n:9.2f} us avg  x{n // args.iters}/fwd  {100 * ms / args.iters / tot:5.1f}%")


if __name__ == "__main__":
    main()
