"""Per-layer precision plans and quantization-site naming.

Same modes, per-layer precisions, prefix-sweep shape and site names as the
reference (reference: pkg/src/samp/encoder.py:44-136), plus one extension the
north star names and the reference lacks: ``MHA_ONLY`` (INT8 attention block,
floating-point FFN).  Its sites are the attention sites plus ``ffn.in``; its
numerics are defined by composition (reference ``mha_int8`` then
``dequantize(ffn.in)`` then ``ffn_fp``, encoder.py:333-385 and :315-330) and
are flagged as an extension wherever reported.
"""

from __future__ import annotations

import functools

from dataclasses import dataclass

from .errors import ConfigurationError

FP = "FP"
FULLY_QUANT = "FULLY_QUANT"
FFN_ONLY = "FFN_ONLY"
MHA_ONLY = "MHA_ONLY"               # extension

LAYER_FP = "FP"
LAYER_FFN_INT8 = "FFN_ONLY_INT8"
LAYER_FULL_INT8 = "FULL_INT8"
LAYER_MHA_INT8 = "MHA_ONLY_INT8"    # extension

_KIND = {FP: LAYER_FP, FULLY_QUANT: LAYER_FULL_INT8, FFN_ONLY: LAYER_FFN_INT8, MHA_ONLY: LAYER_MHA_INT8}
_ALLOWED = {mode: {LAYER_FP, kind} for mode, kind in _KIND.items()}

# C-ABI layer precision codes (include/samp_b200.h SAMP_LAYER_*)
LAYER_CODE = {LAYER_FP: 0, LAYER_FFN_INT8: 1, LAYER_FULL_INT8: 2, LAYER_MHA_INT8: 3}

EMBED_OUT_SITE = "embed.out"
ATTN_NAMES = ("q", "k", "v", "softmax", "out_in")
FFN_NAMES = ("in", "mid")


def attn_in_site(i: int) -> str:
    return f"L{i}.attn.in"


def attn_site(i: int, name: str) -> str:
    return f"L{i}.attn.{name}"


def ffn_site(i: int, name: str) -> str:
    return f"L{i}.ffn.{name}"


def activation_sites(num_layers: int) -> list:
    """All 1 + 8L sites a calibration covers (reference encoder.py:76-83)."""
    out = [EMBED_OUT_SITE]
    for i in range(num_layers):
        out.append(attn_in_site(i))
        out += [attn_site(i, n) for n in ATTN_NAMES]
        out += [ffn_site(i, n) for n in FFN_NAMES]
    return out


@dataclass(frozen=True)
class PrecisionPlan:
    mode: str
    layer_precisions: tuple

    def __post_init__(self):
        if self.mode not in _ALLOWED:
            raise ConfigurationError(f"unknown plan mode {self.mode!r}")
        object.__setattr__(self, "layer_precisions", tuple(self.layer_precisions))
        bad = set(self.layer_precisions) - _ALLOWED[self.mode]
        if bad:
            raise ConfigurationError(f"layer precisions {sorted(bad)} are not allowed in mode {self.mode}")

    @classmethod
    def prefix(cls, mode: str, num_layers: int, quantized: int) -> "PrecisionPlan":
        """First ``quantized`` layers in the mode's INT8 flavour, the rest FP."""
        if not 0 <= quantized <= num_layers:
            raise ConfigurationError(f"quantized layer count {quantized} outside [0, {num_layers}]")
        if mode == FP and quantized > 0:
            raise ConfigurationError("FP mode cannot quantize layers")
        if mode not in _KIND:
            raise ConfigurationError(f"unknown plan mode {mode!r}")
        return cls(mode, tuple(_KIND[mode] if j < quantized else LAYER_FP for j in range(num_layers)))

    @property
    def num_layers(self) -> int:
        return len(self.layer_precisions)

    @property
    def quantized_layer_count(self) -> int:
        return sum(p != LAYER_FP for p in self.layer_precisions)

    def input_site(self, i: int) -> str:
        return EMBED_OUT_SITE if i == 0 else attn_in_site(i)

    def required_sites(self) -> set:
        return set(_required_sites(self.layer_precisions))

    def codes(self) -> bytes:
        """Per-layer precision codes for the C-ABI."""
        return _codes(self.layer_precisions)


@functools.lru_cache(maxsize=256)
def _codes(layer_precisions: tuple) -> bytes:
    return bytes(LAYER_CODE[p] for p in layer_precisions)


@functools.lru_cache(maxsize=256)
def _required_sites(layer_precisions: tuple) -> frozenset:
    """Sites a plan reads (reference encoder.py:126-136); cached per plan (hot per forward)."""
    need = set()
    for i, p in enumerate(layer_precisions):
        if p in (LAYER_FULL_INT8, LAYER_MHA_INT8):
            need.add(EMBED_OUT_SITE if i == 0 else attn_in_site(i))
            need.update(attn_site(i, n) for n in ATTN_NAMES)
            need.add(ffn_site(i, "in"))
            if p == LAYER_FULL_INT8:
                need.add(ffn_site(i, "mid"))
        elif p == LAYER_FFN_INT8:
            need.update((ffn_site(i, "in"), ffn_site(i, "mid")))
    return frozenset(need)
