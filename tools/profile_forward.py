"""Run N forwards of one bench workload configuration (profiling driver for ncu captures).

    python tools/profile_forward.py --workload c2|c4|c5 [--batch B] [--mode FP|FFN_ONLY|FULLY_QUANT]
                                    [--fp16-storage] [--iters N]

Same archive, calibration and synthetic batch as bench.py (batch defaults to the workload's,
e.g. --workload c2 --batch 1 --mode FP --fp16-storage is config C1).  No timing: run it
under ncu with a kernel filter and a launch skip.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--fp16-storage", action="store_true")
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_2209_09130_b200 import _lib
    from paper_2209_09130_b200.engine import HEAD_CLASSIFY, HEAD_TAG, IO_DEVICE, Engine
    from paper_2209_09130_b200.plan import PrecisionPlan
    from paper_2209_09130_b200.tokenization import EncodedInput

    wl = bench.WORKLOADS[args.workload]
    arch = bench.build_model(wl)
    eng = Engine(arch, device=0, fp16_storage=args.fp16_storage)
    L = arch.manifest.num_layers
    if arch.calibration is None:
        c_start, _, c_ids, c_segs = bench.synthetic_batch(1, 8, wl.seq, wl.pairs)
        arch.calibration = eng.calibrate([EncodedInput(c_ids[c_start[i]:c_start[i + 1]].tolist(),
                                                       c_segs[c_start[i]:c_start[i + 1]].tolist(), wl.seq)
                                          for i in range(8)])
        eng._push_calibration()
    mode = args.mode or wl.mode
    codes = PrecisionPlan.prefix(mode, L, 0 if mode == "FP" else L).codes()
    batch = args.batch or wl.batch
    seq_start, att, ids, segs = bench.synthetic_batch(0, batch, wl.seq, wl.pairs)
    dev = torch.device("cuda", 0)
    d_ids, d_segs = torch.from_numpy(ids).to(dev), torch.from_numpy(segs).to(dev)
    head = HEAD_TAG if wl.task == "sequence_labeling" else HEAD_CLASSIFY
    rows = int(seq_start[-1]) if head == HEAD_TAG else batch
    nl = arch.manifest.num_labels
    d_logits = torch.empty((rows, nl), dtype=torch.float32, device=dev)
    d_probs = torch.empty_like(d_logits)
    d_labels = torch.empty(rows, dtype=torch.int32, device=dev)
    lib = _lib.load()
    out = _lib.Outputs(None, d_logits.data_ptr(), d_probs.data_ptr(), d_labels.data_ptr(), head)
    for _ in range(args.iters):
        _lib.check(lib.samp_forward(eng.handle, codes, batch, seq_start.ctypes.data, att.ctypes.data,
                                    d_ids.data_ptr(), d_segs.data_ptr(), IO_DEVICE, out, None))
    torch.cuda.synchronize()
    print(f"done: {args.workload} batch {batch} mode {mode} fp16_storage {args.fp16_storage}, "
          f"{eng.last_launch_count()} launches per forward")


if __name__ == "__main__":
    main()
