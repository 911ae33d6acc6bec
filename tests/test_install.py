"""The drop-in install point, checked on CPU against the real
reference package when it is importable (the build container); no compute."""

from __future__ import annotations

import os
import sys

import pytest

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = next((p for p in ("/root/reference/pkg/src", os.path.join(_ROOT, "baseline", "_ref"))
            if os.path.isdir(os.path.join(p, "tensortune"))), "")


@pytest.fixture
def tensortune():
    if not REF:
        pytest.skip("reference package not present (neither /root/reference nor baseline/_ref)")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import tensortune as tt
    import tensortune.models  # noqa: F401
    import tensortune.sampling  # noqa: F401
    import tensortune.transfer  # noqa: F401

    return tt


def test_install_routes_reference_names_and_uninstall_restores(tensortune):
    import tensortune.models as tm
    import tensortune.sampling as ts
    import tensortune.transfer as tr

    import paper_2304_05430_b200 as pkg
    from paper_2304_05430_b200 import install as inst

    orig = (tm.RecurrentAttentionTuner, tm.CostMLP, tm.pairwise_comparison_accuracy,
            ts.filter_invalid, tr._grouped_pca, tm.per_task_metrics)
    inst.install()
    try:
        assert tm.RecurrentAttentionTuner is pkg.RecurrentAttentionTuner
        assert tm.CostMLP is pkg.CostMLP
        assert tm.pairwise_comparison_accuracy is pkg.pairwise_comparison_accuracy
        assert tr.pairwise_comparison_accuracy is pkg.pairwise_comparison_accuracy
        assert ts.filter_invalid.__module__ == "paper_2304_05430_b200.sampling"
        assert tr._grouped_pca is pkg.grouped_pca
        assert tm.per_task_metrics is not orig[5]
        # load_model / fine_tune resolve the class at call time -> ours
        est, _ = tm._estimator_for("tuner", tm.TrainConfig().to_json())
        assert isinstance(est, pkg.RecurrentAttentionTuner)
        clone = type(est)(**est.get_params())
        assert clone.get_params() == est.get_params()
    finally:
        inst.uninstall()
    assert (tm.RecurrentAttentionTuner, tm.CostMLP, tm.pairwise_comparison_accuracy,
            ts.filter_invalid, tr._grouped_pca, tm.per_task_metrics) == orig


def test_estimator_signatures_match_reference(tensortune):
    import inspect

    from tensortune.estimators import CostMLP as RefMLP
    from tensortune.estimators import RecurrentAttentionTuner as RefTuner

    import paper_2304_05430_b200 as pkg

    for ours, ref in ((pkg.RecurrentAttentionTuner, RefTuner), (pkg.CostMLP, RefMLP)):
        assert inspect.signature(ours.__init__) == inspect.signature(ref.__init__)
        assert ours().get_params() == ref().get_params()
        for meth in ("fit", "predict", "loss_and_gradients", "get_weights", "set_weights"):
            assert list(inspect.signature(getattr(ours, meth)).parameters) == \
                list(inspect.signature(getattr(ref, meth)).parameters), meth
    assert list(inspect.signature(pkg.RecurrentAttentionTuner.continue_fit).parameters) == \
        list(inspect.signature(RefTuner.continue_fit).parameters)
