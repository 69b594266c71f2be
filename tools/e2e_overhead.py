"""Where the e2e step's time goes beyond the device forward (C2, one GPU):
the public forward_packed call (L2 flushed before, as bench.py's e2e) against the same
call with samp_forward replaced by a no-op (Python-side work only) and the device-only
forward (CUDA events on the caller's stream).

    python tools/e2e_overhead.py [--workload c2] [--iters 50]
"""
import argparse
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2209_09130_b200 import _lib  # noqa: E402
from paper_2209_09130_b200.engine import Engine, IO_DEVICE, HEAD_CLASSIFY  # noqa: E402
from paper_2209_09130_b200.plan import PrecisionPlan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    wl = bench.WORKLOADS[args.workload]
    arch = bench.build_model(wl)
    eng = Engine(arch)
    L = arch.manifest.num_layers
    plan = PrecisionPlan.prefix(wl.mode, L, L)
    seq_start, att, ids, segs = bench.workload_batch(wl, 0, 1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def e2e(n, do_flush=True):
        ts = []
        for _ in range(n):
            if do_flush:
                flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.forward_packed(plan, seq_start, att, ids, segs, hidden=False)
            ts.append((time.perf_counter() - t0) * 1e6)
        return statistics.median(ts)

    for _ in range(5):
        eng.forward_packed(plan, seq_start, att, ids, segs, hidden=False)
    full = e2e(args.iters)
    warm = e2e(args.iters, do_flush=False)
    # device-only forward (device ids, caller's stream, events)
    d_ids = torch.from_numpy(ids).cuda()
    d_segs = torch.from_numpy(segs).cuda()
    nl = arch.manifest.num_labels
    B = len(att)
    dl = torch.empty((B, nl), device="cuda")
    dp = torch.empty_like(dl)
    dlab = torch.empty(B, dtype=torch.int32, device="cuda")
    out = _lib.Outputs(None, dl.data_ptr(), dp.data_ptr(), dlab.data_ptr(), HEAD_CLASSIFY)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    lib = _lib.load()
    codes = plan.codes()

    def fwd():
        _lib.check(lib.samp_forward(eng.handle, codes, B, seq_start.ctypes.data, att.ctypes.data,
                                    d_ids.data_ptr(), d_segs.data_ptr(), IO_DEVICE, out, st.cuda_stream))
    for _ in range(5):
        fwd()
    dev = []
    host_dev = []
    for _ in range(args.iters):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        fwd()
        b.record()
        b.synchronize()
        host_dev.append((time.perf_counter() - t0) * 1e6)
        dev.append(a.elapsed_time(b) * 1e3)
    # Python-side only: samp_forward as a no-op
    real = eng._lib.samp_forward

    class Fake:
        def __getattr__(self, k):
            return getattr(real_lib, k)
    real_lib = eng._lib
    eng._lib = Fake()
    eng._lib.__dict__["samp_forward"] = lambda *a: 0
    py = e2e(args.iters, do_flush=False)
    eng._lib = real_lib
    print(f"e2e forward_packed (flushed) {full:.1f} us, warm {warm:.1f} us; device forward {statistics.median(dev):.1f} us "
          f"(host-timed {statistics.median(host_dev):.1f}); Python-side only {py:.1f} us")


if __name__ == "__main__":
    main()
