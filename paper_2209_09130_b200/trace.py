"""Operation tracing for the drop-in API: GEMM / quantize / layer-boundary events.

The reference records these from inside its numpy kernels (reference:
pkg/src/samp/trace.py:1-99, emitted by kernels.py and encoder.py).  On the GPU
the same events are derived from the precision plan and sequence length on
the host — the device kernels are fused, so there is no per-op call to hook —
following the reference's dataflow (encoder.py:472-530) one event at a time.
Tests use them for the dataflow and cost contracts (6 INT8 GEMMs per fully
quantized layer, 2 per FFN-only layer, int8 boundaries between quantized layers).
"""

from __future__ import annotations

import contextlib
from contextvars import ContextVar
from dataclasses import dataclass, field

from .plan import (EMBED_OUT_SITE, LAYER_FFN_INT8, LAYER_FP, LAYER_FULL_INT8, LAYER_MHA_INT8,
                   attn_in_site, attn_site, ffn_site)


@dataclass(frozen=True)
class GemmEvent:
    kind: str      # "f32" or "i8"
    m: int
    k: int
    n: int
    batch: int = 1
    tag: str = ""

    @property
    def bytes_moved(self) -> int:
        width = 4 if self.kind == "f32" else 1
        return self.batch * (width * (self.m * self.k + self.k * self.n) + 4 * self.m * self.n)


@dataclass(frozen=True)
class QuantEvent:
    op: str        # "quantize" | "dequantize" | "requantize"
    site: str


@dataclass(frozen=True)
class BoundaryEvent:
    layer: int
    edge: str      # "enter" | "exit"
    dtype: str     # "f32" | "i8"


@dataclass
class OpTrace:
    gemms: list = field(default_factory=list)
    quant_events: list = field(default_factory=list)
    boundaries: list = field(default_factory=list)

    def gemm_count(self, kind: str) -> int:
        return sum(g.kind == kind for g in self.gemms)

    def gemm_bytes(self, kind: str | None = None) -> int:
        return sum(g.bytes_moved for g in self.gemms if kind is None or g.kind == kind)

    def quant_count(self, op: str, site: str | None = None) -> int:
        return sum(q.op == op and (site is None or q.site == site) for q in self.quant_events)

    def sites(self, op: str) -> list:
        return [q.site for q in self.quant_events if q.op == op]


_CURRENT: ContextVar = ContextVar("samp_b200_trace", default=None)


@contextlib.contextmanager
def trace_ops():
    tr = OpTrace()
    token = _CURRENT.set(tr)
    try:
        yield tr
    finally:
        _CURRENT.reset(token)


def active() -> OpTrace | None:
    return _CURRENT.get()


def record_forward(tr: OpTrace, precisions, seq: int, hidden: int, heads: int, inter: int) -> None:
    """Append the events the reference emits for one Engine.run of a length-`seq` input."""
    d = hidden // heads
    g = tr.gemms.append
    q = lambda op, site: tr.quant_events.append(QuantEvent(op, site))  # noqa: E731

    def attention(kind, i):
        g(GemmEvent(kind, seq, hidden, 3 * hidden, 1, attn_site(i, "qkv")))
        g(GemmEvent(kind, seq, d, seq, heads, attn_site(i, "scores")))
        g(GemmEvent(kind, seq, seq, d, heads, attn_site(i, "context")))
        g(GemmEvent(kind, seq, hidden, hidden, 1, attn_site(i, "out")))

    def ffn(kind, i):
        g(GemmEvent(kind, seq, hidden, inter, 1, ffn_site(i, "w1")))
        g(GemmEvent(kind, seq, inter, hidden, 1, ffn_site(i, "w2")))

    L = len(precisions)
    state_i8, state_site = False, ""
    for i, prec in enumerate(precisions):
        tr.boundaries.append(BoundaryEvent(i, "enter", "i8" if state_i8 else "f32"))
        if prec in (LAYER_FP, LAYER_FFN_INT8):
            if state_i8:
                q("dequantize", state_site)
                state_i8 = False
            attention("f32", i)
            if prec == LAYER_FP:
                ffn("f32", i)
            else:
                q("quantize", ffn_site(i, "in"))
                ffn("i8", i)
                q("quantize", ffn_site(i, "mid"))
        else:
            if not state_i8:
                state_site = EMBED_OUT_SITE if i == 0 else attn_in_site(i)
                q("quantize", state_site)
                state_i8 = True
            attention("i8", i)
            for name in ("q", "k", "v", "softmax", "out_in"):
                q("quantize", attn_site(i, name))
            q("quantize", ffn_site(i, "in"))
            if prec == LAYER_MHA_INT8:     # extension: FP FFN on dequantized ffn.in
                q("dequantize", ffn_site(i, "in"))
                ffn("f32", i)
                state_i8 = False
            else:
                ffn("i8", i)
                q("quantize", ffn_site(i, "mid"))
                nxt = i + 1 < L and precisions[i + 1] in (LAYER_FULL_INT8, LAYER_MHA_INT8)
                if nxt:
                    state_site = attn_in_site(i + 1)
                    q("quantize", state_site)
                else:
                    state_i8 = False
        tr.boundaries.append(BoundaryEvent(i, "exit", "i8" if state_i8 else "f32"))
    if state_i8:
        q("dequantize", state_site)
