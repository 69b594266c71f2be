"""Batch-1 latency with a cold L2 (256 MiB flush before each forward), a warm L2 (no flush),
and cold + the L2 weight prefetch (SAMP_PREFETCH=1): is the small-batch forward HBM-bound?

    python tools/l2_probe.py [--mode FP|FULLY_QUANT] [--fp16-storage]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="FULLY_QUANT")
    ap.add_argument("--fp16-storage", action="store_true")
    ap.add_argument("--iters", type=int, default=30)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2209_09130_b200 import _lib
    from paper_2209_09130_b200.engine import HEAD_CLASSIFY, IO_DEVICE, Engine
    from paper_2209_09130_b200.plan import PrecisionPlan

    arch = bench.build_model()
    eng = Engine(arch, device=0, fp16_storage=args.fp16_storage)
    L = arch.manifest.num_layers
    codes = PrecisionPlan.prefix(args.mode, L, 0 if args.mode == "FP" else L).codes()
    seq_start, att, ids, segs = bench.synthetic_batch(0, 1, 128)
    dev = torch.device("cuda", 0)
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))   # not the legacy default stream (0 = engine's own)
    d_ids, d_segs = torch.from_numpy(ids).to(dev), torch.from_numpy(segs).to(dev)
    d_out = torch.empty((3, 2), dtype=torch.float32, device=dev)
    lib = _lib.load()
    out = _lib.Outputs(None, d_out[0].data_ptr(), d_out[1].data_ptr(), d_out[2].data_ptr(), HEAD_CLASSIFY)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)

    def fwd():
        _lib.check(lib.samp_forward(eng.handle, codes, 1, seq_start.ctypes.data, att.ctypes.data, d_ids.data_ptr(),
                                    d_segs.data_ptr(), IO_DEVICE, out, torch.cuda.current_stream(dev).cuda_stream))

    def run(cold):
        ts = []
        for _ in range(args.iters):
            if cold:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fwd()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    for _ in range(5):
        fwd()
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fwd()
    torch.cuda.synchronize()
    print(f"launches per forward {eng.last_launch_count()}, wall {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms/forward")
    cold = run(True)
    warm = run(False)
    os.environ["SAMP_PREFETCH"] = "1"
    for _ in range(3):
        fwd()
    cold_pf = run(True)
    warm_pf = run(False)
    print(f"{args.mode} fp16_storage={args.fp16_storage}: cold {cold:.4f} ms, warm {warm:.4f} ms, "
          f"cold+prefetch {cold_pf:.4f} ms, warm+prefetch {warm_pf:.4f} ms")


if __name__ == "__main__":
    main()
