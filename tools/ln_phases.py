"""Sub-phases of the LayerNorm GEMM epilogue (register-resident variant) from in-kernel stamps.

    python tools/ln_phases.py [--batch 32]

Per LN GEMM kind (out-proj, FFN2), mean over CTAs: accumulator ready -> x formed (TMEM
read, dequant, bias, residual), leaf sum, row-sum exchange (half + cluster), variance leaf,
variance exchange + rsqrt, normalise + quantize + store.
"""
import argparse
import ctypes
import os
import sys
from collections import defaultdict

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--mode", default="FULLY_QUANT")
    ap.add_argument("--fp16-storage", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2209_09130_b200 import _lib
    from paper_2209_09130_b200.engine import HEAD_CLASSIFY, IO_DEVICE, Engine
    from paper_2209_09130_b200.plan import PrecisionPlan

    arch = bench.build_model()
    eng = Engine(arch, device=0, fp16_storage=args.fp16_storage)
    L = arch.manifest.num_layers
    codes = PrecisionPlan.prefix(args.mode, L, 0 if args.mode == "FP" else L).codes()
    seq_start, att, ids, segs = bench.synthetic_batch(0, args.batch, 128)
    dev = torch.device("cuda", 0)
    d_ids, d_segs = torch.from_numpy(ids).to(dev), torch.from_numpy(segs).to(dev)
    d_logits = torch.empty((args.batch, 2), dtype=torch.float32, device=dev)
    d_probs = torch.empty_like(d_logits)
    d_labels = torch.empty(args.batch, dtype=torch.int32, device=dev)
    lib = _lib.load()
    out = _lib.Outputs(None, d_logits.data_ptr(), d_probs.data_ptr(), d_labels.data_ptr(), HEAD_CLASSIFY)

    def fwd():
        _lib.check(lib.samp_forward(eng.handle, codes, args.batch, seq_start.ctypes.data, att.ctypes.data,
                                    d_ids.data_ptr(), d_segs.data_ptr(), IO_DEVICE, out, None))

    for _ in range(3):
        fwd()
    _lib.check(lib.samp_set_profiling(eng.handle, 1))
    nmax = 8 * L
    _lib.check(lib.samp_debug_gemm_stamps(eng.handle, nmax))
    fwd()
    fwd()
    _lib.check(lib.samp_debug_gemm_stamps(eng.handle, nmax))
    fwd()
    buf = np.zeros((nmax, 1024, 8), np.uint64)
    names = ctypes.create_string_buffer(1 << 14)
    n = ctypes.c_int(0)
    _lib.check(lib.samp_debug_gemm_stamps_fetch(eng.handle, buf.ctypes.data, nmax, names, len(names),
                                                 ctypes.byref(n)))
    names = names.value.decode().split("\n")[: n.value]
    agg = defaultdict(list)
    for i, name in enumerate(names):
        if name not in ("outproj_i8", "ffn2_i8", "outproj_f16", "ffn2_f16"):
            continue
        st = buf[i].astype(np.int64)
        for b in range(512):
            main, sub = st[b], st[512 + b]
            if main[4] == 0 or sub[0] == 0 or sub[5] == 0:
                continue
            agg[name].append([sub[0] - main[4], sub[1] - sub[0], sub[2] - sub[1], sub[3] - sub[2],
                              sub[4] - sub[3], sub[5] - sub[4], main[5] - sub[5]])
    lab = ["form_x", "leaf_sum", "xchg_sum", "leaf_var", "xchg_var", "emit", "tail"]
    for name, rows in agg.items():
        m = np.mean(np.array(rows, np.float64), 0) / 1e3
        print(f"{name:12s} n={len(rows)}  " + "  ".join(f"{l}={v:.2f}" for l, v in zip(lab, m)) + f"  total={m.sum():.2f} us")


if __name__ == "__main__":
    main()
