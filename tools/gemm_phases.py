"""Per-phase timing of the encoder GEMMs from in-kernel %globaltimer stamps.

    python tools/gemm_phases.py [--batch 32] [--seq 128] [--mode FULLY_QUANT]

Runs the bench workload once with GEMM stamps on (profiling mode, no graphs) and prints,
per GEMM kind (averaged over layers): kernel span, CTAs, CTAs per SM at once, and the
mean per-CTA phases: launch->first slot full (pipeline fill), first->last slot full
(main loop loads), last full->accumulator done (MMA drain), epilogue, teardown.
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
    ap.add_argument("--seq", type=int, default=128)
    ap.add_argument("--mode", default="FULLY_QUANT")
    args = ap.parse_args()
    import torch
    from paper_2209_09130_b200 import _lib
    from paper_2209_09130_b200.engine import HEAD_CLASSIFY, IO_DEVICE, Engine
    from paper_2209_09130_b200.plan import PrecisionPlan

    arch = bench.build_model()
    eng = Engine(arch, device=0)
    L = arch.manifest.num_layers
    codes = PrecisionPlan.prefix(args.mode, L, 0 if args.mode == "FP" else L).codes()
    seq_start, att, ids, segs = bench.synthetic_batch(0, args.batch, args.seq)
    dev = torch.device("cuda", 0)
    d_ids, d_segs = torch.from_numpy(ids).to(dev), torch.from_numpy(segs).to(dev)
    nl = arch.manifest.num_labels
    d_logits = torch.empty((args.batch, nl), dtype=torch.float32, device=dev)
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
    fwd()   # second pass: warm instruction caches / TMA descriptors
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
        st = buf[i].astype(np.int64)
        st = st[st[:, 1] != 0]
        t0 = st[:, 1].min()
        att = name.startswith("attention")
        end = 7 if att else 6     # attention: stamp 7 = exit (1 start, 2 S ready, 3-6 softmax passes)
        span = (st[:, end].max() - t0) / 1e3
        ph = np.stack([st[:, j + 1] - st[:, j] for j in range(1, end)], 1) / 1e3
        # residency: max CTAs of this launch alive on one SM at the same time
        per_sm = defaultdict(list)
        for row in st:
            per_sm[int(row[0])].append((row[1], row[end]))
        conc = 0
        for iv in per_sm.values():
            ev = sorted([(a, 1) for a, _ in iv] + [(b, -1) for _, b in iv], key=lambda x: (x[0], x[1]))
            c = m = 0
            for _, d in ev:
                c += d
                m = max(m, c)
            conc = max(conc, m)
        last_start = (st[:, 1].max() - t0) / 1e3
        agg[name].append((span, len(st), len(per_sm), conc, last_start, ph.mean(0), ph.max(0)))
    print(f"{'gemm':12s} {'span_us':>8s} {'ctas':>5s} {'sms':>4s} {'conc':>4s} {'lastst':>7s} | "
          f"{'fill':>6s} {'loads':>6s} {'drain':>6s} {'epi':>6s} {'tear':>6s}  (mean per CTA, us; max in [])")
    print(f"{'':52s}attention phases: load+MMA1, pass1, pass2, sum, pass3, MMA2+out")
    for name, rows in agg.items():
        span = np.mean([r[0] for r in rows])
        ph = np.mean([r[5] for r in rows], 0)
        mx = np.mean([r[6] for r in rows], 0)
        r0 = rows[0]
        print(f"{name:12s} {span:8.2f} {r0[1]:5d} {r0[2]:4d} {r0[3]:4d} {np.mean([r[4] for r in rows]):7.2f} | "
              + " ".join(f"{v:6.2f}" for v in ph) + "  [" + " ".join(f"{v:.1f}" for v in mx) + "]")


if __name__ == "__main__":
    main()
