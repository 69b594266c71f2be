"""Per-item phase timeline of the fused QKV+attention kernel from in-kernel stamps.

    python tools/qa_phases.py [--batch 32] [--seq 128]

Prints, averaged over the fused launches of one FULLY_QUANT forward (CTAs < 128, items < 4),
per item slot: GEMM issue time, QKV epilogue time, softmax passes (pass 1, pass 2, sum,
pass 3), MMA-2 wait, ctx store, and the gaps between them (all microseconds), plus the
kernel span (first stamp -> last ctx store).
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--seq", type=int, default=128)
    args = ap.parse_args()
    import torch
    from paper_2209_09130_b200 import _lib
    from paper_2209_09130_b200.engine import HEAD_CLASSIFY, IO_DEVICE, Engine
    from paper_2209_09130_b200.plan import PrecisionPlan

    arch = bench.build_model()
    eng = Engine(arch, device=0)
    L = arch.manifest.num_layers
    codes = PrecisionPlan.prefix("FULLY_QUANT", L, L).codes()
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
    fwd()
    _lib.check(lib.samp_debug_gemm_stamps(eng.handle, nmax))
    fwd()
    buf = np.zeros((nmax, 1024, 8), np.uint64)
    names = ctypes.create_string_buffer(1 << 14)
    n = ctypes.c_int(0)
    _lib.check(lib.samp_debug_gemm_stamps_fetch(eng.handle, buf.ctypes.data, nmax, names, len(names),
                                                 ctypes.byref(n)))
    names = names.value.decode().split("\n")[: n.value]
    rows = []
    for i, name in enumerate(names):
        if name != "qkv_attention_i8":
            continue
        st = buf[i].reshape(128, 4, 16).astype(np.int64)
        t0 = st[:, :, [0, 10]][st[:, :, [0, 10]] > 0].min()
        rows.append((st, t0))
    print(f"{len(rows)} fused launches")
    labels = ["gemm", "epi_wait", "epi", "->soft", "pass1", "pass2", "sum", "pass3", "o_wait", "ctx"]
    for j in range(4):
        vals = []
        for st, t0 in rows:
            for b in range(128):
                r = st[b, j]
                if r[9] == 0:
                    continue
                vals.append([r[11] - r[10], r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[5] - r[4],
                             r[6] - r[5], r[7] - r[6], r[8] - r[7], r[9] - r[8], r[10] - t0, r[9] - t0])
        if not vals:
            continue
        v = np.array(vals, np.float64) / 1e3
        m = v.mean(0)
        print(f"item {j}: n={len(v)}  " + "  ".join(f"{l}={x:.2f}" for l, x in zip(labels, m)) +
              f"  | gemm_start={m[10]:.2f} ctx_done={m[11]:.2f} (max {v[:, 11].max():.2f})")
    names = ["epi_wait", "acc_ready", "epi_done", "soft_start", "pass1", "pass2", "sum", "p_done", "o_ready",
             "ctx_done", "gemm_issue", "gemm_issued", "mma1_issued", "ctx_last", "epi_last", "mma2_issued"]
    print("absolute (us after the CTA's first stamp), mean over CTAs:")
    for j in range(4):
        vals = []
        for st, t0 in rows:
            for b in range(128):
                r = st[b, j]
                if r[9] == 0:
                    continue
                b0 = st[b, 0][st[b, 0] > 0].min()
                vals.append([(x - b0) / 1e3 if x else np.nan for x in r[:16]])
        if vals:
            m = np.nanmean(np.array(vals), 0)
            print(f"item {j}: " + "  ".join(f"{n}={v:.2f}" for n, v in zip(names, m)))
    spans = [(st[:, :, 9].max() - t0) / 1e3 for st, t0 in rows]
    print(f"span: mean {np.mean(spans):.2f} us")


if __name__ == "__main__":
    main()
