"""Probe: do two half-batches on two streams (two engines) beat one full batch?

    python tools/two_stream_probe.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2209_09130_b200 import _lib  # noqa: E402
from paper_2209_09130_b200.engine import HEAD_CLASSIFY, IO_DEVICE, Engine  # noqa: E402
from paper_2209_09130_b200.plan import PrecisionPlan  # noqa: E402


def main():
    arch = bench.build_model()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    plan = PrecisionPlan.prefix("FULLY_QUANT", 12, 12).codes()
    engines = [Engine(arch), Engine(arch)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def setup(B):
        ss, att, ids, segs = bench.synthetic_batch(0, B, 128)
        d_ids, d_segs = torch.from_numpy(ids).to(dev), torch.from_numpy(segs).to(dev)
        lg = torch.empty((B, 2), device=dev)
        pr = torch.empty_like(lg)
        lb = torch.empty(B, dtype=torch.int32, device=dev)
        out = _lib.Outputs(None, lg.data_ptr(), pr.data_ptr(), lb.data_ptr(), HEAD_CLASSIFY)
        return ss, att, d_ids, d_segs, out, (lg, pr, lb)

    def fwd(eng, st, B, cfg):
        ss, att, d_ids, d_segs, out, _ = cfg
        _lib.check(lib.samp_forward(eng.handle, plan, B, ss.ctypes.data, att.ctypes.data, d_ids.data_ptr(),
                                    d_segs.data_ptr(), IO_DEVICE, out, st.cuda_stream))

    for B, n_eng in ((32, 1), (16, 2), (64, 1), (32, 2)):
        cfgs = [setup(B) for _ in range(n_eng)]
        for _ in range(5):
            for i in range(n_eng):
                fwd(engines[i], streams[i], B, cfgs[i])
        torch.cuda.synchronize()
        steps = 20
        tot = 0.0
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(n_eng):
                fwd(engines[i], streams[i], B, cfgs[i])
            torch.cuda.synchronize()
            tot += time.perf_counter() - t0
        sent = B * n_eng * steps / tot
        print(f"batch {B} x {n_eng} engine(s)/streams: {sent:.0f} sentences/s ({tot / steps * 1e3:.3f} ms per step)")


if __name__ == "__main__":
    main()
