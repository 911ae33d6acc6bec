"""Search-time batched scoring on the GPU: the reference's
``tune`` with the GPU tuner scoring one candidate per call, against the
cross-task batched ``tune`` (paper_2304_05430_b200.search) -- identical
TuneResult, far fewer predict calls."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = next((p for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")
            if os.path.isdir(os.path.join(p, "tensortune"))), "")


@pytest.fixture(scope="module")
def gpu_model():
    if not REF:
        pytest.skip("baseline/_ref not staged (tools/stage_reference.py, run by build())")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import tensortune.cli  # noqa: F401
    from tensortune.benchmarks import convergence_benchmark
    from tensortune.features import encode_sequence_batch
    from tensortune.models import CostModel, TrainConfig
    from tensortune.oracle import OracleConfig, oracle_cost

    from paper_2304_05430_b200 import RecurrentAttentionTuner

    ds, a = convergence_benchmark(seed=1, n_tasks=12, records_per_task=40)
    seqs, y = encode_sequence_batch(ds, sorted(a.train_ids))
    est = RecurrentAttentionTuner(epochs=3, seed=0, recurrent_layers=2).fit(seqs, y)
    model = CostModel(kind="tuner", estimator=est, config=TrainConfig(epochs=3, recurrent_layers=2))
    ocfg = OracleConfig(noise_sigma=0.05, seed=0)
    return ds, model, (lambda k, s, hw: oracle_cost(k, s, hw, ocfg))


@pytest.mark.parametrize("method,precision", [("anneal", "fp32"), ("evolve", "fp32"), ("anneal", "tf32")])
def test_batched_tune_identical_to_reference_tune_on_gpu(cuda_ok, gpu_model, method, precision):
    import tensortune.models as tm
    import tensortune.search as ts

    from paper_2304_05430_b200 import _lib
    from paper_2304_05430_b200 import search as bs

    ds, model, oracle_fn = gpu_model
    model.estimator.precision = precision
    tids = [t.task_id for t in ds.tasks]
    cfg = ts.SearchConfig(method=method, steps=96, population=16, generations=4, top_k=4, seed=5)
    bs.bind_reference()
    before = _lib.CALLS.copy()
    want = ts.tune(ds, tids, lambda t: tm.make_schedule_scorer(model, ds.task_by_id[t], ds), oracle_fn, cfg)
    mid = _lib.CALLS.copy()
    got = bs.tune(ds, tids, lambda t: bs.make_schedule_scorer(model, ds.task_by_id[t], ds), oracle_fn, cfg)
    after = _lib.CALLS.copy()
    model.estimator.precision = None
    assert got.to_json() == want.to_json()
    n_ref = sum((mid - before).values())
    n_bat = sum((after - mid).values())
    assert got.scoring_stats["predict_calls"] == n_bat
    assert n_bat * 4 < n_ref, (n_bat, n_ref)  # >= 4x fewer launches (12 tasks per batch at most)
    assert np.isfinite(got.total_best_cost)
