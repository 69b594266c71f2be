"""ctypes binding of libsamp_b200.so (include/samp_b200.h).

Loads the in-tree library built by ``_build.build()``.  There is no CPU
fallback: if the library is missing or the device is not a B200 the calls
raise ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

_PKG = os.path.dirname(os.path.abspath(__file__))
# SAMP_B200_LIB: load another build of the same ABI (A/B timing of kernel variants)
LIB_PATH = os.environ.get("SAMP_B200_LIB") or os.path.join(_PKG, "lib", "libsamp_b200.so")

SAMP_OK = 0
_STATUS = {
    1: errors.DimensionError,
    2: errors.ConfigurationError,
    3: errors.CalibrationError,
    4: errors.InputError,
    5: errors.DeviceError,
    6: errors.EngineError,
}

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_f32p = ctypes.POINTER(ctypes.c_float)


class ModelDesc(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("hidden", ctypes.c_int32), ("num_heads", ctypes.c_int32),
                ("intermediate", ctypes.c_int32), ("vocab_size", ctypes.c_int32),
                ("max_position", ctypes.c_int32), ("type_vocab_size", ctypes.c_int32),
                ("num_labels", ctypes.c_int32), ("layernorm_eps", ctypes.c_double),
                ("fp16_storage", ctypes.c_int32)]


class Outputs(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_void_p), ("logits", ctypes.c_void_p), ("probs", ctypes.c_void_p),
                ("labels", ctypes.c_void_p), ("head", ctypes.c_int32)]


# (name, restype, argtypes) for every symbol in include/samp_b200.h
SIGNATURES = [
    ("samp_last_error", ctypes.c_char_p, []),
    ("samp_device_check", ctypes.c_int, [ctypes.c_int]),
    ("samp_engine_create", ctypes.c_int, [ctypes.POINTER(ModelDesc), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    ("samp_engine_destroy", None, [ctypes.c_void_p]),
    ("samp_load_embeddings", ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_void_p] * 5),
    ("samp_load_layer", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    ("samp_load_heads", ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_void_p] * 4),
    ("samp_weight_scales", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    ("samp_set_site_amax", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_double]),
    ("samp_clear_calibration", ctypes.c_int, [ctypes.c_void_p]),
    ("samp_forward", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int32, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                    ctypes.POINTER(Outputs), ctypes.c_void_p]),
    ("samp_calibrate", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]),
    ("samp_code_usage", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int32, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("samp_set_exact_fp32", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("samp_set_graphs", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("samp_sync", ctypes.c_int, [ctypes.c_void_p]),
    ("samp_set_capture", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("samp_fetch_stage", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    ("samp_debug_gemm_i8", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("samp_debug_gemm_f16", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("samp_debug_gemm_peak", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.POINTER(ctypes.c_float)]),
    ("samp_debug_quant_exhaustive", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong)]),
    ("samp_debug_div_exhaustive", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong)]),
    ("samp_debug_exp_exhaustive", ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong)]),
    ("samp_debug_gelu_finite_exhaustive", ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong)]),
    ("samp_tokenizer_create", ctypes.c_void_p, [ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int]),
    ("samp_tokenizer_destroy", None, [ctypes.c_void_p]),
    ("samp_tokenize_batch", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_char_p),
                                           ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("samp_debug_exp2_fast_exhaustive", ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong)]),
    ("samp_debug_gelu_fast_check", ctypes.c_int, [ctypes.c_float, ctypes.POINTER(ctypes.c_ulonglong)]),
    ("samp_debug_unary", ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]),
    ("samp_last_launch_count", ctypes.c_int, [ctypes.c_void_p]),
    ("samp_set_profiling", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("samp_profile_report", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]),
    ("samp_debug_gemm_stamps", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("samp_debug_gemm_stamps_fetch", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                                     ctypes.c_char_p, ctypes.c_size_t, ctypes.c_void_p]),
]

_lib = None


def load(required=True):
    """Load the library (raises DeviceError when missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not required:
            return None
        raise errors.DeviceError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().samp_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status != SAMP_OK:
        raise _STATUS.get(status, errors.EngineError)(last_error())


def ptr(arr) -> int:
    return arr.ctypes.data
