"""Search-time batched scoring (paper_2304_05430_b200.search)
on the host: cross-task batched ``tune`` returns exactly the reference's
``tune`` result.  The model here is the reference's own GBDT (its predict is
a per-row tree walk, so it is batch invariant like the GPU kernels), which
isolates the batching logic; the GPU version is in
tests/test_gpu_search_batched.py."""

from __future__ import annotations

import os
import sys

import pytest

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = next((p for p in ("/root/reference/pkg/src", os.path.join(_ROOT, "baseline", "_ref"))
            if os.path.isdir(os.path.join(p, "tensortune"))), "")


@pytest.fixture(scope="module")
def setup():
    if not REF:
        pytest.skip("reference package not present")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import tensortune.cli  # noqa: F401
    from tensortune.benchmarks import convergence_benchmark
    from tensortune.models import GBDTConfig, train_gbdt
    from tensortune.oracle import OracleConfig, oracle_cost

    ds, a = convergence_benchmark(seed=0, n_tasks=6, records_per_task=40)
    model, _ = train_gbdt(ds, a, GBDTConfig(num_trees=20))
    ocfg = OracleConfig(noise_sigma=0.05, seed=0)
    return ds, model, (lambda k, s, hw: oracle_cost(k, s, hw, ocfg))


@pytest.mark.parametrize("method", ["anneal", "evolve"])
def test_batched_tune_equals_reference_tune(setup, method):
    import tensortune.models as tm
    import tensortune.search as ts

    from paper_2304_05430_b200 import search as bs

    ds, model, oracle_fn = setup
    tids = [t.task_id for t in ds.tasks]
    cfg = ts.SearchConfig(method=method, steps=48, population=12, generations=4, top_k=4, seed=3)
    bs.bind_reference()
    want = ts.tune(ds, tids, lambda t: tm.make_schedule_scorer(model, ds.task_by_id[t], ds), oracle_fn, cfg)
    got = bs.tune(ds, tids, lambda t: bs.make_schedule_scorer(model, ds.task_by_id[t], ds), oracle_fn, cfg,
                  jobs=3)
    assert got.to_json() == want.to_json()
    st = got.scoring_stats
    # each predict call carried several tasks' candidates
    assert 0 < st["predict_calls"] < st["programs"]
    if method == "anneal":
        assert st["predict_calls"] <= cfg.steps + 1


def test_unbatchable_scorers_fall_back_to_the_reference(setup):
    import numpy as np
    import tensortune.search as ts

    from paper_2304_05430_b200 import search as bs

    ds, _, oracle_fn = setup
    tids = [t.task_id for t in ds.tasks][:3]
    cfg = ts.SearchConfig(method="anneal", steps=20, top_k=2, seed=1)

    def factory(tid):
        return lambda schedules: np.array([float(sum(s.tile_factors[0])) for s in schedules])

    bs.bind_reference()
    assert bs.tune(ds, tids, factory, oracle_fn, cfg).to_json() == \
        ts.tune(ds, tids, factory, oracle_fn, cfg).to_json()
