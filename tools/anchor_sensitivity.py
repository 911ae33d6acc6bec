"""How much does the reference's own 200-epoch val rmse move under a
rounding-level perturbation?  Generates tests/golden/anchor_sensitivity.jsonl,
the anchor band of tests/anchors/anchor_convergence.py.

Runs the UNMODIFIED reference (CPU, float64; test_acceptance.py:174-195's
configuration: convergence_benchmark(seed), TrainConfig(epochs=200,
learning_rate=1e-3, recurrent_layers=2, seed=seed)) with every initial
weight multiplied by (1 + eps): eps = 0 is the reference as shipped; eps of
a few 1e-15 is a few ulps, the size of the difference between two correct
float64 implementations of the same arithmetic (summation order, libm).

    PYTHONPATH=baseline/_ref OPENBLAS_NUM_THREADS=1 \\
        python tools/anchor_sensitivity.py SEED EPS >> tests/golden/anchor_sensitivity.jsonl

(one process per (seed, eps); ~8 minutes each on one core.)
"""

from __future__ import annotations

import json
import sys
import time

from tensortune.benchmarks import convergence_benchmark
from tensortune.estimators import tuner as ref_tuner
from tensortune.models import TrainConfig, train_tuner

seed, eps = int(sys.argv[1]), float(sys.argv[2])
_orig_init = ref_tuner.RecurrentAttentionTuner._init_params


def _perturbed_init(self):
    _orig_init(self)
    for v in self.params_.values():
        v *= 1.0 + eps


ref_tuner.RecurrentAttentionTuner._init_params = _perturbed_init
ds, a = convergence_benchmark(seed=seed)
t = time.time()
_, rep = train_tuner(ds, a, TrainConfig(epochs=200, learning_rate=1e-3, recurrent_layers=2, seed=seed))
print(json.dumps({"seed": seed, "eps": eps, "val_rmse": rep.val_rmse, "wall_s": round(time.time() - t, 1)}),
      flush=True)
