"""GPU-side knobs, kept out of the reference's TrainConfig (models.py:66-107)
so model files stay byte-compatible.

PRECISION: "fp32" (production: float32 kernels, stated tolerances) or
"fp64" (the same kernels instantiated in float64: parity/debug build, lets
the reference's finite-difference gradient checks run against the GPU).
Override per estimator with ``est.precision = "fp64"`` or globally with the
TT_PRECISION environment variable.
"""

from __future__ import annotations

import os

PRECISION = os.environ.get("TT_PRECISION", "fp32")

# Largest minibatch a single fused training launch accepts (one CTA per
# sample up to the SM count, more samples per CTA beyond it).
MAX_BATCH = 4096
