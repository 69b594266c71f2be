"""Cross-kernel timeline of one forward (PDL chain as in a normal run, no graph, no events):
per stamped launch the first CTA start, the first real work (first operand stage landed /
first GEMM issue) and the last CTA's end, in µs from the forward's first stamp, plus the gap
from each kernel's end to the next one's first work.

    python tools/timeline.py [--batch 32] [--mode FP|FULLY_QUANT] [--layers 2]

Caveat: stamps need direct launches (no CUDA graph), so the gaps here include the host's
launch submission; the graph-launched forward's gaps are the SAMP_SKIP critical-path costs
minus the spans (tools/skip_b1.sh, tools/skip_ab.sh).  (The persistent FFN1 kernel keeps a
per-tile stamp layout and shows no span here.)
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
    ap.add_argument("--mode", default="FULLY_QUANT")
    ap.add_argument("--layers", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2209_09130_b200 import _lib
    from paper_2209_09130_b200.engine import HEAD_CLASSIFY, IO_DEVICE, Engine
    from paper_2209_09130_b200.plan import PrecisionPlan

    arch = bench.build_model()
    eng = Engine(arch, device=0)
    L = arch.manifest.num_layers
    codes = PrecisionPlan.prefix(args.mode, L, 0 if args.mode == "FP" else L).codes()
    seq_start, att, ids, segs = bench.synthetic_batch(0, args.batch, 128)
    dev = torch.device("cuda", 0)
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))
    d_ids, d_segs = torch.from_numpy(ids).to(dev), torch.from_numpy(segs).to(dev)
    d_out = torch.empty((3, args.batch, 2), dtype=torch.float32, device=dev)
    lib = _lib.load()
    out = _lib.Outputs(None, d_out[0].data_ptr(), d_out[1].data_ptr(), d_out[2].data_ptr(), HEAD_CLASSIFY)

    def fwd():
        _lib.check(lib.samp_forward(eng.handle, codes, args.batch, seq_start.ctypes.data, att.ctypes.data,
                                    d_ids.data_ptr(), d_segs.data_ptr(), IO_DEVICE, out,
                                    torch.cuda.current_stream(dev).cuda_stream))

    for _ in range(3):
        fwd()
    nmax = 8 * L
    _lib.check(lib.samp_set_profiling(eng.handle, 2))
    _lib.check(lib.samp_debug_gemm_stamps(eng.handle, nmax))
    fwd()
    fwd()
    _lib.check(lib.samp_debug_gemm_stamps(eng.handle, nmax))
    fwd()
    torch.cuda.synchronize()
    _lib.check(lib.samp_set_profiling(eng.handle, 0))
    buf = np.zeros((nmax, 1024, 8), np.uint64)
    names = ctypes.create_string_buffer(1 << 14)
    n = ctypes.c_int(0)
    _lib.check(lib.samp_debug_gemm_stamps_fetch(eng.handle, buf.ctypes.data, nmax, names, len(names),
                                                 ctypes.byref(n)))
    names = names.value.decode().split("\n")[: n.value]
    rows = []
    for i, name in enumerate(names):
        st = buf[i].astype(np.int64)
        if name.startswith("qkv_attention"):
            r = st.reshape(128, 4, 16)
            starts = r[:, :, 10][r[:, :, 10] > 0]
            ends = np.concatenate([r[:, :, 9][r[:, :, 9] > 0], r[:, :, 13][r[:, :, 13] > 0]])
            if not len(starts):
                continue
            rows.append((name, starts.min(), starts.min(), ends.max()))
        else:
            live = st[:512]
            live = live[live[:, 1] > 0]
            if not len(live):
                continue
            end_col = 7 if name.startswith("attention") else 6
            work = live[:, 2][live[:, 2] > 0]
            rows.append((name, live[:, 1].min(), work.min() if len(work) else live[:, 1].min(), live[:, end_col].max()))
    t0 = min(r[1] for r in rows)
    print(f"{'kernel':20s} {'start':>8s} {'work':>8s} {'end':>8s} {'span':>7s} {'gap_to_next_work':>17s}")
    for k, (name, a, w, e) in enumerate(rows[: 4 * args.layers + 1]):
        gap = (rows[k + 1][2] - e) / 1e3 if k + 1 < len(rows) else float("nan")
        print(f"{name:20s} {(a - t0) / 1e3:8.2f} {(w - t0) / 1e3:8.2f} {(e - t0) / 1e3:8.2f} {(e - w) / 1e3:7.2f} {gap:17.2f}")


if __name__ == "__main__":
    main()
