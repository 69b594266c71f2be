"""B200-native SAMP (arXiv 2209.09130): self-adaptive mixed-precision BERT encoder.

Drop-in for the reference ``samp`` package's hot path: same archive/scale layout,
``Engine``/``PrecisionPlan`` API, heads and sweep tooling; the encoder forward runs
in hand-written sm_100a kernels (libsamp_b200.so).
"""

from .archive import ModelArchive, ModelManifest, load_archive, write_archive
from .errors import (CalibrationError, ConfigurationError, DeviceError, DimensionError, EngineError,
                     InputError)
from .plan import FFN_ONLY, FP, FULLY_QUANT, MHA_ONLY, PrecisionPlan
from .quantization import (CalibrationTable, CodeUsageReport, QuantScale, code_usage, dequantize,
                           minmax_observe, quantize, requantize_i32)
from .tokenization import EncodedInput, Vocab, encode, tokenize

__version__ = "0.1.0"


def __getattr__(name):
    # device-backed pieces import lazily so host-only tooling works without a GPU
    if name in ("Engine", "EncoderOutput", "BatchOutput"):
        from . import engine
        return getattr(engine, name)
    if name in ("classify", "tag", "match", "TaskResult"):
        from . import tasks
        return getattr(tasks, name)
    if name in ("Profile", "ProfilePoint", "allocate_decay_aware", "build_profile", "rank_by_ratio",
                "select_by_accuracy_threshold", "select_by_latency_threshold"):
        from . import allocator
        return getattr(allocator, name)
    if name in ("trace_ops",):
        from . import trace
        return trace.trace_ops
    raise AttributeError(name)


__all__ = [
    "CalibrationTable", "CodeUsageReport", "EncodedInput", "EncoderOutput", "Engine", "FFN_ONLY", "FP",
    "FULLY_QUANT", "MHA_ONLY", "ModelArchive", "ModelManifest", "PrecisionPlan", "Profile", "ProfilePoint",
    "QuantScale", "TaskResult", "Vocab", "allocate_decay_aware", "build_profile", "classify", "code_usage",
    "dequantize", "encode", "load_archive", "match", "minmax_observe", "quantize", "rank_by_ratio",
    "requantize_i32", "select_by_accuracy_threshold", "select_by_latency_threshold", "tag", "tokenize",
    "write_archive", "BatchOutput", "CalibrationError", "ConfigurationError", "DeviceError",
    "DimensionError", "EngineError", "InputError",
]
