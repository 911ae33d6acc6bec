"""How much does the reference's own 200-epoch val rmse move under a
rounding-level perturbation?  (Context for the convergence-anchor tolerance,
tests/anchors/anchor_convergence.py.)

Runs the UNMODIFIED reference (CPU, float64) on convergence_benchmark(seed)
twice per seed: as shipped, and with every initial weight multiplied by
(1 + 1e-15) -- a few ulps, the size of the difference between two correct
float64 implementations (summation order, libm ulps).  Prints JSON lines.

    PYTHONPATH=baseline/_ref OPENBLAS_NUM_THREADS=1 python tools/anchor_sensitivity.py
"""

from __future__ import annotations

import json
import sys
import time

import numpy as np
from tensortune.benchmarks import convergence_benchmark
from tensortune.estimators import tuner as ref_tuner
from tensortune.models import TrainConfig, train_tuner

_orig_init = ref_tuner.RecurrentAttentionTuner._init_params


def _perturbed_init(self):
    _orig_init(self)
    for v in self.params_.values():
        v *= 1.0 + 1e-15


seeds = [int(a) for a in sys.argv[1:]] or [0, 1, 2]
for seed in seeds:
    for perturb in (False, True):
        ref_tuner.RecurrentAttentionTuner._init_params = _perturbed_init if perturb else _orig_init
        ds, a = convergence_benchmark(seed=seed)
        t = time.time()
        _, rep = train_tuner(ds, a, TrainConfig(epochs=200, learning_rate=1e-3, recurrent_layers=2,
                                                seed=seed))
        print(json.dumps({"seed": seed, "perturbed_1e-15": perturb, "val_rmse": rep.val_rmse,
                          "wall_s": round(time.time() - t, 1)}), flush=True)
