"""How ill-conditioned are FFN_ONLY logits in the reference itself?  (CPU, oracle only)

    python tools/ffn_only_conditioning.py [--n 48] [perturbation ...]

Runs BERT-base (bench weights + reference calibration), FFN_ONLY k=12 at S=128 on the
oracle twice — once as the reference computes it, once with the attention block perturbed —
and prints the relative change of the classification logits.  Perturbations:
  f64   one change only: each layer's QKV GEMM accumulated in float64 and rounded once,
        instead of the reference's k-ordered float32 (a ~1e-7 relative change)
  w     f16-rounded weights of the attention GEMMs        x    f16-rounded GEMM inputs
  qkv   f16-rounded q/k/v                                  p    f16-rounded probabilities
  ctx   f16-rounded context
Measured (build container, 48 sequences): f64 4.9%, w 10.7%, x 10.9%, qkv 10.3%, p 11.1%.
Twelve rounds of quantize(ffn.in) -> INT8 FFN turn any perturbation into code flips that
compound, so no implementation that is not bit-identical can meet a 1e-2 logits tolerance
on this plan; Engine(exact_fp32=True) is bit-identical (tests/test_gpu_exact_fp32.py).
The oracle's GEMMs run as BLAS sgemm here (oracle.blas_fp32) for speed: the baseline and
the perturbed run share it, so only the named perturbation differs.
"""

from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import samp_oracle as orc  # noqa: E402

F32 = np.float32


def h16(x):
    return np.asarray(x, F32).astype(np.float16).astype(F32)


def make_mha(which):
    def mha(mm, i, x, att_len, taps=None, rnd=None):
        h = mm.hidden
        d = h // mm.num_heads
        W = (lambda k: h16(mm.lw(i, k))) if "w" in which else (lambda k: mm.lw(i, k))
        xin = h16(x) if "x" in which else x
        qkv_w = np.concatenate([W("qw"), W("kw"), W("vw")], axis=1)
        qkv_b = np.concatenate([mm.lw(i, "qb"), mm.lw(i, "kb"), mm.lw(i, "vb")])
        if "f64" in which:
            qkv = ((xin.astype(np.float64) @ qkv_w.astype(np.float64)).astype(F32) + qkv_b).astype(F32)
        else:
            qkv = (orc.gemm_f32(xin, qkv_w) + qkv_b).astype(F32)
        if "qkv" in which:
            qkv = h16(qkv)
        q, k, v = qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:]
        qh, kh, vh = orc._split(q, mm.num_heads), orc._split(k, mm.num_heads), orc._split(v, mm.num_heads)
        sc = np.stack([orc.gemm_f32(qh[a], kh[a].T.copy()) for a in range(mm.num_heads)])
        sc = sc * F32(1.0 / math.sqrt(d)) + orc._mask(x.shape[0], att_len)
        p = orc.softmax(sc.astype(F32))
        if "p" in which:
            p = h16(p)
        ctx = orc._merge(np.stack([orc.gemm_f32(p[a], vh[a]) for a in range(mm.num_heads)]))
        if "ctx" in which:
            ctx = h16(ctx)
        proj = orc.gemm_f32(ctx, W("ow"))
        return orc.layernorm(((proj + mm.lw(i, "ob")) + x).astype(F32), mm.lw(i, "ln1_g"), mm.lw(i, "ln1_b"),
                             mm.eps)
    return mha


def main():
    from paper_2209_09130_b200.quantization import CalibrationTable
    from paper_2209_09130_b200.synthetic import bert_archive
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=48)
    ap.add_argument("which", nargs="*", default=["f64"])
    args = ap.parse_args()
    arch = bert_archive("bert-base")
    with open(os.path.join(ROOT, "tests", "golden", "bench_calibration_bert-base.json")) as fh:
        table = CalibrationTable.from_json(fh.read())
    model = orc.Model.from_manifest(arch.manifest, arch.tensors, {s: e.amax for s, e in table.entries.items()})
    ids = np.random.default_rng(1234).integers(0, 30522, size=(args.n, 128))
    plan = orc.plan_prefix("FFN_ONLY", 12, 12)
    base_mha = orc.mha_fp
    with orc.blas_fp32():
        ref = np.array([orc.classify_logits(model, orc.run(model, r, [0] * 128, 128, plan))[0] for r in ids])
        for w in args.which:
            orc.mha_fp = make_mha(w.split(","))
            try:
                got = np.array([orc.classify_logits(model, orc.run(model, r, [0] * 128, 128, plan))[0] for r in ids])
            finally:
                orc.mha_fp = base_mha
            print(f"{w}: logits relative change {np.linalg.norm(got - ref) / np.linalg.norm(ref):.4f}")


if __name__ == "__main__":
    main()
