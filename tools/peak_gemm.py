"""Measured tensor peaks for the roofline denominators (run under gpurun, one B200).

    python tools/peak_gemm.py [--out profiles/peaks_int8_f16.json]

* INT8 dense: cuBLASLt through torch._int_mm, 8192^3 int8 x int8 -> int32 (2*N^3 ops):
  best of 10 launches (burst, for a kernel timed alone) and back to back for 4 s
  (sustained, under the power cap).
* FP16 dense: torch.matmul f16 8192^3, the same two ways (MEASURED_PEAKS.json has bf16).
* This repo's own tcgen05 GEMM main loop (kind::i8 / kind::f16, plain accumulator store,
  samp_debug_gemm_peak) at the same size: the ceiling of the main loop the fused kernels
  are built on.
Clocks are sampled with nvidia-smi during each sustained loop.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _clock_sampler():
    return subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                             "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                            stderr=subprocess.DEVNULL, text=True)


def _stop(p):
    p.terminate()
    out = p.communicate()[0]
    sm = []
    for line in out.splitlines():
        try:
            sm.append(float(line.split(",")[0]))
        except ValueError:
            pass
    return statistics.median(sm) if sm else None


def _measure(fn, ops):
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    clk = _clock_sampler()
    n, t0 = 0, time.time()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    b.record()
    b.synchronize()
    sus_ms = a.elapsed_time(b) / n
    sm = _stop(clk)
    return {"burst_tops": round(ops / (best * 1e-3) / 1e12, 1), "sustained_tops": round(ops / (sus_ms * 1e-3) / 1e12, 1),
            "burst_ms": round(best, 4), "sustained_ms": round(sus_ms, 4), "sm_mhz_median_sustained": sm}


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "peaks_int8_f16.json"))
    args = ap.parse_args()
    N = args.n
    ops = 2.0 * N ** 3
    dev = torch.device("cuda", 0)
    res = {"n": N, "ops_per_launch": ops, "gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    a8 = torch.randint(-128, 127, (N, N), dtype=torch.int8, device=dev)
    b8 = torch.randint(-128, 127, (N, N), dtype=torch.int8, device=dev).t().contiguous().t()
    res["int8_cublaslt"] = _measure(lambda: torch._int_mm(a8, b8), ops)
    res["int8_cublaslt"]["how"] = "torch._int_mm (cuBLASLt) int8 x int8 -> int32"
    del a8, b8
    ah = torch.randn(N, N, dtype=torch.float16, device=dev)
    bh = torch.randn(N, N, dtype=torch.float16, device=dev)
    res["f16_cublas"] = _measure(lambda: torch.matmul(ah, bh), ops)
    res["f16_cublas"]["how"] = "torch.matmul f16 (cuBLAS), f32 accumulate"
    del ah, bh
    torch.cuda.empty_cache()
    from paper_2209_09130_b200 import _lib
    lib = _lib.load()
    for kind, name in ((0, "int8_own_tcgen05"), (1, "f16_own_tcgen05")):
        ms = ctypes.c_float()
        _lib.check(lib.samp_debug_gemm_peak(kind, N, N, N, 3, ctypes.byref(ms)))
        _lib.check(lib.samp_debug_gemm_peak(kind, N, N, N, 20, ctypes.byref(ms)))
        res[name] = {"tops": round(ops / (ms.value * 1e-3) / 1e12, 1), "ms": round(ms.value, 4),
                     "how": "gemm_kernel<BN=256, 4 stages, one 128-row tile per CTA> + EpiStoreAcc, 20 launches"}
    print(json.dumps(res, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
