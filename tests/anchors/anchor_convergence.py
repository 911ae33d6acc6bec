"""End-to-end parity anchor for GPU training.

Run only under tests/refsuite_plugin.py (the reference's ``tensortune`` with
``install()`` applied), by tests/test_gpu_reference_suite.py.

The reference's acceptance check (test_acceptance.py:174-195) trains the
tuner for 200 epochs on convergence_benchmark(seed) and asks val rmse <= 0.06
and <= GBDT.  The exact 200-epoch value is a chaotic function of rounding:
the unmodified reference ITSELF, with its initial weights scaled by
(1 + eps) for eps in {1e-15, -1e-15, 2e-15} (a few ulps), lands anywhere in
0.0358-0.0473 for seed 2 (tests/golden/anchor_sensitivity.jsonl, made by
tools/anchor_sensitivity.py).  So the anchor is that ensemble: a GPU-trained
tuner must land inside [ensemble min - 0.005, ensemble max + 0.005] of the
reference's own ulp-perturbation runs for its seed, under 0.06, and below the
reference GBDT's val rmse on the same split (0.0767 / 0.0863 / 0.0886,
SURVEY.md §6.3).
"""

from __future__ import annotations

import json
import os

import pytest
from tensortune.benchmarks import convergence_benchmark
from tensortune.models import TrainConfig, train_tuner

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURE = os.path.join(os.path.dirname(HERE), "golden", "anchor_sensitivity.jsonl")
REF_GBDT_VAL_RMSE = {0: 0.0767, 1: 0.0863, 2: 0.0886}
MARGIN = 0.005


def _ensemble(seed):
    with open(FIXTURE) as fh:
        rows = [json.loads(x) for x in fh if x.strip()]
    return sorted(r["val_rmse"] for r in rows if r["seed"] == seed)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tuner_200_epoch_val_rmse_inside_reference_ensemble(seed):
    ens = _ensemble(seed)
    assert len(ens) >= 3
    ds, assignment = convergence_benchmark(seed=seed)
    model, rep = train_tuner(
        ds, assignment, TrainConfig(epochs=200, learning_rate=1e-3, recurrent_layers=2, seed=seed))
    assert type(model.estimator).__module__.startswith("paper_2304_05430_b200")
    lo, hi = ens[0] - MARGIN, ens[-1] + MARGIN
    print(f"seed {seed}: GPU val rmse {rep.val_rmse:.4f}; reference ensemble "
          f"{', '.join(f'{v:.4f}' for v in ens)} -> band [{lo:.4f}, {hi:.4f}]; gbdt {REF_GBDT_VAL_RMSE[seed]:.4f}")
    assert lo <= rep.val_rmse <= hi, rep.val_rmse
    assert rep.val_rmse <= 0.06
    assert rep.val_rmse <= REF_GBDT_VAL_RMSE[seed]
