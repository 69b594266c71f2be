"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's mixed-precision encoder forward
(reference: pkg/src/samp/encoder.py, kernels.py, quantization.py, tasks.py).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it and has no CPU
fallback.

Arithmetic follows the reference operation by operation (float32 numpy
elementwise ops, numpy's pairwise float32 reductions, INT8 GEMMs exact through
float64).  The two float32 transcendentals are routed through
``oracle/npmath.c`` — a bit-exact restatement of numpy's own ``np.exp`` and
(SVML) ``np.tanh`` — so the oracle reproduces the reference's numbers on any
host CPU, including hosts whose numpy would dispatch to a different SIMD
kernel.

Parity is pinned against the real reference imported in the build container:
``tests/golden/make_golden.py`` regenerates fixtures from the reference and
``tests/test_oracle.py`` checks this module against them bit-for-bit.

Structure (each stage is a pure function of its inputs so GPU stage outputs
can be teacher-forced through it):
  embed                        encoder.py:249-273
  qkv_int8 / attention_int8 /
  out_proj_int8                encoder.py:333-385 (mha_int8)
  ffn1_int8 / ffn2_int8        encoder.py:388-418 (ffn_int8)
  mha_fp / ffn_fp              encoder.py:276-330
  run                          encoder.py:472-530 (Engine.run dispatch)
  classify / tag               tasks.py:28-55
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
I8 = np.int8
I32 = np.int32

HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(HERE, "_build")
_LIB_PATH = os.path.join(_BUILD, "libnpmath.so")

AMAX_FLOOR = 127 * 1e-8                     # quantization.py:24-25
MASK_VALUE = F32(-10000.0)                   # encoder.py:61
_GELU_C = F32(math.sqrt(2.0 / math.pi))     # kernels.py:29
_GELU_K = F32(0.044715)                      # kernels.py:30

LAYER_FP = "FP"
LAYER_FFN = "FFN_ONLY_INT8"
LAYER_FULL = "FULL_INT8"
LAYER_MHA = "MHA_ONLY_INT8"                  # extension: no reference counterpart


# ----------------------------------------------------------------- npmath lib

def build_npmath(force: bool = False) -> str:
    """Compile oracle/npmath.c (gcc, no FP contraction) into oracle/_build."""
    src = os.path.join(HERE, "npmath.c")
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src):
        return _LIB_PATH
    os.makedirs(_BUILD, exist_ok=True)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
                    "-o", _LIB_PATH, src, "-lm"], check=True)
    return _LIB_PATH


_lib = None


def _npmath():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_npmath())
        for fn in (_lib.npm_exp_array, _lib.npm_tanh_array):
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]
            fn.restype = None
    return _lib


def _apply(fn_name: str, x: np.ndarray) -> np.ndarray:
    src = np.ascontiguousarray(x, dtype=F32)
    out = np.empty_like(src)
    getattr(_npmath(), fn_name)(src.ctypes.data, out.ctypes.data, src.size)
    return out


def np_exp(x):
    """Bit-exact restatement of numpy float32 exp."""
    return _apply("npm_exp_array", x)


def np_tanh(x):
    """Bit-exact restatement of numpy float32 tanh (SVML)."""
    return _apply("npm_tanh_array", x)


# ----------------------------------------------------------------- primitives

def site_scale(amax: float) -> float:
    """QuantScale.scale (quantization.py:78-80): double arithmetic."""
    return float(max(float(amax), AMAX_FLOOR) / 127.0)


def quantize(x, scale: float) -> np.ndarray:
    """quantization.py:33-39 — trunc(x/s + copysign(.5)), clip, int8."""
    y = np.asarray(x, dtype=F32) / F32(scale)
    q = np.trunc(y + np.copysign(F32(0.5), y))
    return np.clip(q, -128, 127).astype(I8)


def dequant(q, scale: float) -> np.ndarray:
    """quantization.py:42-47 / encoder._deq_codes: F32(q) * F32(s)."""
    return (q.astype(F32) * F32(scale)).astype(F32)


def deq_acc(acc, sa: float, sb: float) -> np.ndarray:
    """encoder._deq_acc (encoder.py:228-231): one F32 multiplier from a double product."""
    return (acc.astype(F32) * F32(float(sa) * float(sb))).astype(F32)


def gemm_i8(a, b) -> np.ndarray:
    """kernels.gemm_i8_i32 (kernels.py:112-127): exact via float64."""
    return (a.astype(np.float64) @ b.astype(np.float64)).astype(I32)


def gemm_f32(a, b) -> np.ndarray:
    """kernels._gemm_f32_fast (kernels.py:62-71): rank-1 updates, k order, no FMA."""
    out = np.zeros((a.shape[0], b.shape[1]), dtype=F32)
    for t in range(a.shape[1]):
        out += a[:, t:t + 1] * b[t:t + 1, :]
    return out


class blas_fp32:
    """Context manager for large-sample STATISTICAL tests only: the FP32 GEMMs run as BLAS
    sgemm instead of the reference's rank-1 k-order loop (kernels.py:62-71).  Results then
    differ from the reference by float32 summation order (~1e-6 relative), far inside the
    FP16-path tolerance those tests check; every bit-exact test keeps the restatement.
    exp / tanh are numpy's own here (the npmath restatement is only needed for bit-exact
    parity on hosts whose numpy dispatches differently)."""

    def __enter__(self):
        global gemm_f32, np_exp, np_tanh
        self._saved = gemm_f32, np_exp, np_tanh
        gemm_f32 = lambda a, b: np.matmul(np.asarray(a, F32), np.asarray(b, F32)).astype(F32)  # noqa: E731
        # numpy's own float32 transcendentals (== npmath on the AVX512 hosts it restates)
        np_exp = lambda x: np.exp(np.asarray(x, F32))    # noqa: E731
        np_tanh = lambda x: np.tanh(np.asarray(x, F32))  # noqa: E731
        return self

    def __exit__(self, *exc):
        global gemm_f32, np_exp, np_tanh
        gemm_f32, np_exp, np_tanh = self._saved


def softmax(x) -> np.ndarray:
    """kernels.softmax_rows (kernels.py:130-135)."""
    shifted = x - np.max(x, axis=-1, keepdims=True)
    e = np_exp(shifted)
    return (e / np.sum(e, axis=-1, keepdims=True)).astype(F32)


def layernorm(x, gamma, beta, eps: float) -> np.ndarray:
    """kernels.layernorm (kernels.py:138-154): numpy pairwise means."""
    mean = np.mean(x, axis=-1, keepdims=True, dtype=F32)
    c = x - mean
    var = np.mean(c * c, axis=-1, keepdims=True, dtype=F32)
    inv = F32(1.0) / np.sqrt(var + F32(eps))
    return (c * inv * gamma + beta).astype(F32)


def gelu(x) -> np.ndarray:
    """kernels.gelu (kernels.py:157-161), tanh form."""
    inner = _GELU_C * (x + _GELU_K * x * x * x)
    return (F32(0.5) * x * (F32(1.0) + np_tanh(inner))).astype(F32)


def f16_round(x) -> np.ndarray:
    return np.asarray(x, dtype=F32).astype(np.float16).astype(F32)


def pairwise_sum(a: np.ndarray) -> np.float32:
    """numpy's float32 pairwise reduction, restated (used to pin the GPU tree).

    n < 8: sequential from 0; n <= 128: 8 strided accumulators combined
    ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then a sequential tail; larger n
    splits at n/2 rounded down to a multiple of 8.  np.sum adds the result
    to an initial 0.
    """
    def rec(lo, n):
        if n < 8:
            r = F32(0.0)
            for i in range(n):
                r = F32(r + a[lo + i])
            return r
        if n <= 128:
            r = [F32(a[lo + j]) for j in range(8)]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] = F32(r[j] + a[lo + i + j])
                i += 8
            res = F32(F32(F32(r[0] + r[1]) + F32(r[2] + r[3])) + F32(F32(r[4] + r[5]) + F32(r[6] + r[7])))
            while i < n:
                res = F32(res + a[lo + i])
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return F32(rec(lo, n2) + rec(lo + n2, n - n2))

    return F32(F32(0.0) + rec(0, len(a)))


# ----------------------------------------------------------------- model

def layer_key(i: int, name: str) -> str:
    """archive.layer_keys (archive.py:95-106)."""
    p = f"encoder.layer.{i}"
    table = {
        "qw": "attn.q.weight", "qb": "attn.q.bias", "kw": "attn.k.weight", "kb": "attn.k.bias",
        "vw": "attn.v.weight", "vb": "attn.v.bias", "ow": "attn.out.weight", "ob": "attn.out.bias",
        "ln1_g": "attn.layernorm.gamma", "ln1_b": "attn.layernorm.beta",
        "w1": "ffn.w1", "b1": "ffn.b1", "w2": "ffn.w2", "b2": "ffn.b2",
        "ln2_g": "ffn.layernorm.gamma", "ln2_b": "ffn.layernorm.beta",
    }
    return f"{p}.{table[name]}"


def weight_quant(w: np.ndarray):
    """encoder.quantize_weight (encoder.py:191-194): per-tensor, scale from max|w|."""
    s = site_scale(float(np.max(np.abs(w))))
    return quantize(w, s), s


@dataclass
class QLayer:
    qkv: np.ndarray            # [H, 3H] int8 (blocks q|k|v, separately scaled)
    s_qkv: tuple
    wo: np.ndarray
    s_wo: float
    w1: np.ndarray
    s_w1: float
    w2: np.ndarray
    s_w2: float


@dataclass
class Model:
    """Manifest fields + F32 tensors (archive layout) + calibration amax."""

    num_layers: int
    hidden: int
    num_heads: int
    intermediate: int
    eps: float
    tensors: dict
    amax: dict = field(default_factory=dict)
    fp16_storage: bool = False
    task: str = "classification"
    _q: dict = field(default_factory=dict)

    @classmethod
    def from_manifest(cls, manifest, tensors, amax=None, fp16_storage=False):
        g = (lambda k: manifest[k]) if isinstance(manifest, dict) else (lambda k: getattr(manifest, k))
        return cls(g("num_layers"), g("hidden"), g("num_heads"), g("intermediate"),
                   float(g("layernorm_eps")), tensors, dict(amax or {}), fp16_storage, g("task"))

    def t(self, key):
        return self.tensors[key]

    def lw(self, i, name):
        return self.tensors[layer_key(i, name)]

    def scale(self, site):
        return site_scale(self.amax[site])

    def qlayer(self, i) -> QLayer:
        """QuantizedLayerWeights.from_f32 (encoder.py:210-225)."""
        if i not in self._q:
            qq, sq = weight_quant(self.lw(i, "qw"))
            kq, sk = weight_quant(self.lw(i, "kw"))
            vq, sv = weight_quant(self.lw(i, "vw"))
            oq, so = weight_quant(self.lw(i, "ow"))
            q1, s1 = weight_quant(self.lw(i, "w1"))
            q2, s2 = weight_quant(self.lw(i, "w2"))
            self._q[i] = QLayer(np.ascontiguousarray(np.concatenate([qq, kq, vq], axis=1)),
                                (sq, sk, sv), oq, so, q1, s1, q2, s2)
        return self._q[i]


def _site(i, block, name):
    return f"L{i}.{block}.{name}"


def _mask(seq: int, att_len: int) -> np.ndarray:
    m = np.zeros(seq, dtype=F32)
    m[att_len:] = MASK_VALUE
    return m


def _split(x, heads):
    s, h = x.shape
    return np.ascontiguousarray(x.reshape(s, heads, h // heads).transpose(1, 0, 2))


def _merge(x):
    a, s, d = x.shape
    return np.ascontiguousarray(x.transpose(1, 0, 2).reshape(s, a * d))


# ----------------------------------------------------------------- stages

def embed(m: Model, ids, segs):
    """encoder.embed_fused (encoder.py:249-273), F32 result before storage rounding."""
    ids = np.asarray(ids)
    segs = np.asarray(segs)
    summed = (m.t("embeddings.word.weight")[ids] + m.t("embeddings.position.weight")[: len(ids)]) \
        + m.t("embeddings.token_type.weight")[segs]
    return layernorm(summed.astype(F32), m.t("embeddings.layernorm.gamma"),
                     m.t("embeddings.layernorm.beta"), m.eps)


def qkv_int8(m: Model, i, x_q, s_in):
    """encoder.py:355-366: fused QKV INT8 GEMM, per-block dequant + bias, quantize."""
    ql = m.qlayer(i)
    h = m.hidden
    acc = gemm_i8(x_q, ql.qkv)
    outs = []
    for blk, (nm, bias) in enumerate((("q", "qb"), ("k", "kb"), ("v", "vb"))):
        f = deq_acc(acc[:, blk * h:(blk + 1) * h], s_in, ql.s_qkv[blk]) + m.lw(i, bias)
        outs.append(f)
    codes = [quantize(f, m.scale(_site(i, "attn", nm))) for f, nm in zip(outs, "qkv")]
    return acc, outs, codes


def attention_int8(m: Model, i, q_c, k_c, v_c, att_len):
    """encoder.py:368-379: per-head INT8 scores, masked softmax, INT8 context."""
    d = m.hidden // m.num_heads
    s_q, s_k, s_v = (m.scale(_site(i, "attn", n)) for n in "qkv")
    s_sm = m.scale(_site(i, "attn", "softmax"))
    s_ctx = m.scale(_site(i, "attn", "out_in"))
    qh, kh, vh = _split(q_c, m.num_heads), _split(k_c, m.num_heads), _split(v_c, m.num_heads)
    score_acc = gemm_i8(qh, kh.transpose(0, 2, 1))
    scores = score_acc.astype(F32) * F32(s_q * s_k / math.sqrt(d))
    scores = scores + _mask(q_c.shape[0], att_len)
    probs = softmax(scores.astype(F32))
    probs_q = quantize(probs, s_sm)
    ctx_acc = gemm_i8(probs_q, vh)
    ctx = _merge(deq_acc(ctx_acc, s_sm, s_v))
    return dict(score_acc=score_acc, probs=probs, probs_q=probs_q, ctx_acc=ctx_acc,
                ctx=ctx, ctx_q=quantize(ctx, s_ctx))


def out_proj_int8(m: Model, i, ctx_q, x_q, s_in):
    """encoder.py:353,381-385: out-proj GEMM + bias + residual + LN + quantize(ffn.in)."""
    ql = m.qlayer(i)
    residual = dequant(x_q, s_in)
    acc = gemm_i8(ctx_q, ql.wo)
    proj = deq_acc(acc, m.scale(_site(i, "attn", "out_in")), ql.s_wo)
    out = layernorm((proj + m.lw(i, "ob")) + residual, m.lw(i, "ln1_g"), m.lw(i, "ln1_b"), m.eps)
    return acc, out, quantize(out, m.scale(_site(i, "ffn", "in")))


def ffn1_int8(m: Model, i, x_q):
    """encoder.py:406-410: W1 GEMM + dequant + bias + GELU + quantize(ffn.mid)."""
    ql = m.qlayer(i)
    acc = gemm_i8(x_q, ql.w1)
    mid = deq_acc(acc, m.scale(_site(i, "ffn", "in")), ql.s_w1) + m.lw(i, "b1")
    act = gelu(mid.astype(F32))
    return acc, act, quantize(act, m.scale(_site(i, "ffn", "mid")))


def ffn2_int8(m: Model, i, act_q, x_q, out_site=None):
    """encoder.py:405,412-418: W2 GEMM + bias + residual + LN (+ quantize at out_site)."""
    ql = m.qlayer(i)
    residual = dequant(x_q, m.scale(_site(i, "ffn", "in")))
    acc = gemm_i8(act_q, ql.w2)
    y = deq_acc(acc, m.scale(_site(i, "ffn", "mid")), ql.s_w2)
    out = layernorm((y + m.lw(i, "b2")) + residual, m.lw(i, "ln2_g"), m.lw(i, "ln2_b"), m.eps)
    codes = quantize(out, m.scale(out_site)) if out_site else None
    return acc, out, codes


def mha_fp(m: Model, i, x, att_len, taps=None, rnd=None):
    """encoder.mha_fp (encoder.py:276-312)."""
    post = rnd if rnd is not None else (lambda v: v)
    h = m.hidden
    d = h // m.num_heads
    qkv_w = np.ascontiguousarray(np.concatenate([m.lw(i, "qw"), m.lw(i, "kw"), m.lw(i, "vw")], axis=1))
    qkv_b = np.concatenate([m.lw(i, "qb"), m.lw(i, "kb"), m.lw(i, "vb")])
    qkv = post((gemm_f32(x, qkv_w) + qkv_b).astype(F32))
    q, k, v = qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:]
    if taps is not None:
        for nm, val in zip("qkv", (q, k, v)):
            taps[_site(i, "attn", nm)] = np.array(val, dtype=F32)
    qh, kh, vh = _split(q, m.num_heads), _split(k, m.num_heads), _split(v, m.num_heads)
    scores = np.stack([gemm_f32(qh[a], kh[a].T.copy()) for a in range(m.num_heads)])
    scores = scores * F32(1.0 / math.sqrt(d)) + _mask(x.shape[0], att_len)
    probs = post(softmax(scores.astype(F32)))
    if taps is not None:
        taps[_site(i, "attn", "softmax")] = np.array(probs, dtype=F32)
    ctx = post(_merge(np.stack([gemm_f32(probs[a], vh[a]) for a in range(m.num_heads)])))
    if taps is not None:
        taps[_site(i, "attn", "out_in")] = np.array(ctx, dtype=F32)
    proj = gemm_f32(ctx, m.lw(i, "ow"))
    out = post(layernorm(((proj + m.lw(i, "ob")) + x).astype(F32), m.lw(i, "ln1_g"), m.lw(i, "ln1_b"), m.eps))
    if taps is not None:
        taps[_site(i, "ffn", "in")] = np.array(out, dtype=F32)
    return out


def ffn_fp(m: Model, i, x, taps=None, rnd=None):
    """encoder.ffn_fp (encoder.py:315-330)."""
    post = rnd if rnd is not None else (lambda v: v)
    mid = gemm_f32(x, m.lw(i, "w1")) + m.lw(i, "b1")
    act = post(gelu(mid.astype(F32)))
    if taps is not None:
        taps[_site(i, "ffn", "mid")] = np.array(act, dtype=F32)
    y = gemm_f32(act, m.lw(i, "w2"))
    return post(layernorm(((y + m.lw(i, "b2")) + x).astype(F32), m.lw(i, "ln2_g"), m.lw(i, "ln2_b"), m.eps))


def input_site(i):
    return "embed.out" if i == 0 else f"L{i}.attn.in"


def run(m: Model, ids, segs, att_len, layers, taps=None, stages=None):
    """Engine.run dispatch (encoder.py:472-530), plus the MHA-only extension.

    ``layers`` is the per-layer precision tuple.  ``stages`` (a dict) collects
    every intermediate INT8 code / INT32 accumulator for teacher-forced checks.
    """
    rnd = f16_round if m.fp16_storage else None
    hidden = embed(m, ids, segs)
    if rnd is not None:
        hidden = rnd(hidden)
    if taps is not None:
        taps["embed.out"] = np.array(hidden, dtype=F32)
    st = stages if stages is not None else {}
    state_q, state_site = None, ""
    L = len(layers)
    for i, prec in enumerate(layers):
        if prec in (LAYER_FP, LAYER_FFN):
            if state_q is not None:
                hidden = dequant(state_q, m.scale(state_site))
                state_q = None
            if taps is not None:
                taps[f"L{i}.attn.in"] = np.array(hidden, dtype=F32)
            if prec == LAYER_FP:
                hidden = mha_fp(m, i, hidden, att_len, taps, rnd)
                hidden = ffn_fp(m, i, hidden, taps, rnd)
            else:
                mha_out = mha_fp(m, i, hidden, att_len, taps, None)
                x_q = quantize(mha_out, m.scale(_site(i, "ffn", "in")))
                st[f"L{i}.ffn_in_q"] = x_q
                a1, act, act_q = ffn1_int8(m, i, x_q)
                st[f"L{i}.mid_acc"], st[f"L{i}.mid_q"] = a1, act_q
                if taps is not None:
                    taps[_site(i, "ffn", "mid")] = act
                a2, hidden, _ = ffn2_int8(m, i, act_q, x_q, None)
                st[f"L{i}.out_acc"], st[f"L{i}.out"] = a2, hidden
            st[f"L{i}.out"] = hidden
            continue
        # INT8 attention block (FULL and MHA-only layers)
        if state_q is None:
            site = input_site(i)
            if site != "embed.out" and taps is not None:
                taps[site] = np.array(hidden, dtype=F32)
            state_q, state_site = quantize(hidden, m.scale(site)), site
        s_in = m.scale(state_site)
        st[f"L{i}.in_q"] = state_q
        acc, qkv_f, (qc, kc, vc) = qkv_int8(m, i, state_q, s_in)
        st[f"L{i}.qkv_acc"] = acc
        st[f"L{i}.q_q"], st[f"L{i}.k_q"], st[f"L{i}.v_q"] = qc, kc, vc
        if taps is not None:
            for nm, val in zip("qkv", qkv_f):
                taps[_site(i, "attn", nm)] = val
        at = attention_int8(m, i, qc, kc, vc, att_len)
        st[f"L{i}.score_acc"], st[f"L{i}.probs_q"] = at["score_acc"], at["probs_q"]
        st[f"L{i}.ctx_acc"], st[f"L{i}.ctx_q"] = at["ctx_acc"], at["ctx_q"]
        if taps is not None:
            taps[_site(i, "attn", "softmax")] = at["probs"]
            taps[_site(i, "attn", "out_in")] = at["ctx"]
        pacc, ln1, x_q = out_proj_int8(m, i, at["ctx_q"], state_q, s_in)
        st[f"L{i}.proj_acc"], st[f"L{i}.ffn_in_q"] = pacc, x_q
        if taps is not None:
            taps[_site(i, "ffn", "in")] = ln1
        if prec == LAYER_MHA:
            # extension: MHA in INT8, FFN in FP on the dequantized ffn.in codes
            hidden = ffn_fp(m, i, dequant(x_q, m.scale(_site(i, "ffn", "in"))), taps, None)
            state_q = None
            st[f"L{i}.out"] = hidden
            continue
        a1, act, act_q = ffn1_int8(m, i, x_q)
        st[f"L{i}.mid_acc"], st[f"L{i}.mid_q"] = a1, act_q
        if taps is not None:
            taps[_site(i, "ffn", "mid")] = act
        nxt = i + 1 < L and layers[i + 1] in (LAYER_FULL, LAYER_MHA)
        out_site = f"L{i + 1}.attn.in" if nxt else None
        a2, out_f, out_q = ffn2_int8(m, i, act_q, x_q, out_site)
        st[f"L{i}.out_acc"] = a2
        if nxt:
            if taps is not None:
                taps[out_site] = out_f
            state_q, state_site = out_q, out_site
            st[f"L{i}.out"] = out_q
        else:
            hidden, state_q = out_f, None
            st[f"L{i}.out"] = hidden
    if state_q is not None:
        hidden = dequant(state_q, m.scale(state_site))
    return hidden.astype(F32)


# ----------------------------------------------------------------- heads

def classify_logits(m: Model, hidden):
    """tasks.classify (tasks.py:28-41): pooled [CLS] -> logits, probs, argmax."""
    pooled = np_tanh((hidden[0:1] @ m.t("pooler.weight") + m.t("pooler.bias")).astype(F32))
    logits = (pooled @ m.t("head.weight") + m.t("head.bias"))[0].astype(F32)
    probs = softmax(logits[None, :])[0]
    return logits, probs, int(np.argmax(probs))


def tag_logits(m: Model, hidden, att_len):
    """tasks.tag (tasks.py:44-55): per-token logits over the non-pad prefix."""
    h = hidden[:att_len]
    logits = (h @ m.t("head.weight") + m.t("head.bias")).astype(F32)
    probs = softmax(logits)
    return logits, probs, [int(np.argmax(r)) for r in probs]


def plan_prefix(mode: str, num_layers: int, k: int):
    """PrecisionPlan.prefix (encoder.py:102-113) incl. the MHA-only extension."""
    kind = {"FP": LAYER_FP, "FULLY_QUANT": LAYER_FULL, "FFN_ONLY": LAYER_FFN, "MHA_ONLY": LAYER_MHA}[mode]
    return tuple(kind if j < k else LAYER_FP for j in range(num_layers))
