"""Per-tile phase timeline of the persistent GEMMs (FFN1) from in-kernel stamps.

    python tools/persist_phases.py [--batch 32] [--workload c4] [--name ffn1_i8]

For the first FFN1 launch of a FULLY_QUANT forward prints, per CTA (first 64), the tile
count and, averaged over its tiles: epilogue wait for the accumulator, epilogue run time,
MMA-side wait for a free accumulator buffer, main-loop (first box -> last MMA issued);
plus the kernel span and each CTA's finish time.
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
    ap.add_argument("--name", default="ffn1_i8")
    ap.add_argument("--workload", default=None, help="a bench.py workload (its model and batch)")
    args = ap.parse_args()
    import torch
    from paper_2209_09130_b200 import _lib
    from paper_2209_09130_b200.engine import HEAD_CLASSIFY, HEAD_TAG, IO_DEVICE, Engine
    from paper_2209_09130_b200.plan import PrecisionPlan

    wl = bench.WORKLOADS[args.workload] if args.workload else None
    arch = bench.build_model(wl) if wl else bench.build_model()
    eng = Engine(arch, device=0)
    L = arch.manifest.num_layers
    if arch.calibration is None:   # as bench.py: on-device calibration of the synthetic model
        from paper_2209_09130_b200.tokenization import EncodedInput
        c_start, _, c_ids, c_segs = bench.synthetic_batch(1, 8, wl.seq, wl.pairs)
        arch.calibration = eng.calibrate([EncodedInput(c_ids[c_start[i]:c_start[i + 1]].tolist(),
                                                       c_segs[c_start[i]:c_start[i + 1]].tolist(), wl.seq)
                                          for i in range(8)])
        eng._push_calibration()
    codes = PrecisionPlan.prefix("FULLY_QUANT", L, L).codes()
    if wl:
        seq_start, att, ids, segs = bench.workload_batch(wl, 0, 1)
        args.batch = len(att)
    else:
        seq_start, att, ids, segs = bench.synthetic_batch(0, args.batch, bench.SEQ)
    tag = wl is not None and wl.task == "sequence_labeling"
    dev = torch.device("cuda", 0)
    d_ids, d_segs = torch.from_numpy(ids).to(dev), torch.from_numpy(segs).to(dev)
    nl = arch.manifest.num_labels
    rows = int(seq_start[-1]) if tag else args.batch
    d_logits = torch.empty((rows, nl), dtype=torch.float32, device=dev)
    d_probs = torch.empty_like(d_logits)
    d_labels = torch.empty(rows, dtype=torch.int32, device=dev)
    lib = _lib.load()
    out = _lib.Outputs(None, d_logits.data_ptr(), d_probs.data_ptr(), d_labels.data_ptr(),
                       HEAD_TAG if tag else HEAD_CLASSIFY)

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
    li = [i for i, nm in enumerate(names) if nm == args.name][1]   # second layer's launch
    st = buf[li].reshape(64, 16, 8).astype(np.int64)
    valid = st[:, :, 1] != 0
    t0 = st[:, :, 5][st[:, :, 5] != 0].min()
    rel = lambda a: (a - t0) / 1e3
    print(f"{args.name} (layer 2): CTAs 0..63")
    ew, er, mw, ml = [], [], [], []
    for b in range(64):
        nt = int(valid[b].sum())
        if nt == 0:
            continue
        row = st[b, :nt]
        ew.append(np.mean(row[:, 1] - row[:, 0]) / 1e3)
        er.append(np.mean(row[:, 2] - row[:, 1]) / 1e3)
        ml.append(np.mean(row[:, 4] - row[:, 3]) / 1e3)
        if b < 4 or b in (28, 29, 63):
            print(f"  cta {b:3d} tiles {nt}  finish {rel(row[-1, 2]):7.2f}  epi-wait " +
                  " ".join(f"{(r[1]-r[0])/1e3:5.2f}" for r in row) + " | epi-run " +
                  " ".join(f"{(r[2]-r[1])/1e3:5.2f}" for r in row) + " | mma-start " +
                  " ".join(f"{rel(r[3]):6.2f}" for r in row) + " | mainloop " +
                  " ".join(f"{(r[4]-r[3])/1e3:5.2f}" for r in row))
    print(f"  mean per tile: epilogue wait {np.mean(ew):.2f} us, epilogue run {np.mean(er):.2f} us, "
          f"main loop {np.mean(ml):.2f} us")
    fin = [rel(st[b, int(valid[b].sum()) - 1, 2]) for b in range(64) if valid[b].any()]
    print(f"  finish: min {min(fin):.2f} max {max(fin):.2f} us after the first box")


if __name__ == "__main__":
    main()
