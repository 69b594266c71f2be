"""``samp.encoder`` drop-in: the reference module's public names on the B200 engine.

Reference code that imports from ``samp.encoder`` (pkg/src/samp/encoder.py:45-87,
:139-142, :421) finds the same names here: the plan modes and layer kinds, the
activation-site helpers, ``PrecisionPlan``, ``EncoderOutput`` and ``Engine`` (device
backed, imported lazily so host-only tooling works without a GPU).  The numpy layer
functions of the reference (``embed_fused``, ``mha_int8`` ...) are the hot path that the
CUDA kernels replace; their restatement lives in ``oracle/`` (test-only).
"""

from __future__ import annotations

import numpy as np

from .plan import (ATTN_NAMES, EMBED_OUT_SITE, FFN_NAMES, FFN_ONLY, FP, FULLY_QUANT, LAYER_FFN_INT8, LAYER_FP,
                   LAYER_FULL_INT8, LAYER_MHA_INT8, MHA_ONLY, PrecisionPlan, activation_sites, attn_in_site,
                   attn_site, ffn_site)

ATTENTION_MASK_VALUE = np.float32(-10000.0)   # reference encoder.py:61


def __getattr__(name):
    if name in ("Engine", "EncoderOutput", "QuantizedLayerWeights", "BatchOutput"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)


__all__ = ["ATTENTION_MASK_VALUE", "ATTN_NAMES", "EMBED_OUT_SITE", "FFN_NAMES", "FFN_ONLY", "FP", "FULLY_QUANT",
           "LAYER_FFN_INT8", "LAYER_FP", "LAYER_FULL_INT8", "LAYER_MHA_INT8", "MHA_ONLY", "PrecisionPlan",
           "activation_sites", "attn_in_site", "attn_site", "ffn_site", "Engine", "EncoderOutput",
           "QuantizedLayerWeights", "BatchOutput"]
