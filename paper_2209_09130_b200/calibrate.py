"""GPU-side calibration and taps (reference Engine.calibrate, encoder.py:446-454).

Placeholder until the amax-tap kernels land: both entry points raise
ConfigurationError so no caller silently gets CPU-computed values.
"""

from __future__ import annotations

from .errors import ConfigurationError


def calibrate_engine(engine, encoded_inputs):
    raise ConfigurationError("GPU calibration is not implemented yet; load a calibration.json "
                             "produced by the reference (or the oracle) into the archive")


def run_with_taps(engine, enc, plan):
    raise ConfigurationError("capture_taps is not implemented on the GPU path yet")
