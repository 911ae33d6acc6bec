"""GBDT on the GPU (csrc/tt_gbdt.cu) against trees, curves and
predictions produced by the reference itself (tests/golden/gbdt.npz) --
bit for bit -- and against the pinned level-wise oracle on larger random
data."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import gbdt as ogbdt

pytestmark = pytest.mark.gpu


def _fit(X, y, Xv, yv, nt, md, lr, ml):
    from paper_2304_05430_b200 import GradientBoostedTrees

    return GradientBoostedTrees(num_trees=nt, max_depth=md, learning_rate=lr,
                                min_samples_leaf=ml).fit(X, y, eval_set=(Xv, yv))


@pytest.mark.parametrize("name", ["conv", "ties", "adjacent", "single", "deep"])
def test_gbdt_matches_reference_golden_bitwise(cuda_ok, name):
    g = golden("gbdt.npz")
    nt, md, lr, ml = g[f"{name}_params"]
    m = _fit(g[f"{name}_X"], g[f"{name}_y"], g[f"{name}_Xv"], g[f"{name}_yv"], int(nt), int(md), float(lr),
             int(ml))
    w = m.get_weights()
    for k in ("base", "n_features", "node_counts", "feature", "threshold", "left", "right", "value"):
        assert w[k].dtype == g[f"{name}_w_{k}"].dtype, k
        assert np.array_equal(w[k], g[f"{name}_w_{k}"]), (name, k)
    curve = np.array([[a, np.nan if b is None else b] for a, b in m.train_curve_])
    assert np.array_equal(curve, g[f"{name}_curve"], equal_nan=True)
    assert np.array_equal(m.predict(g[f"{name}_Xv"]), g[f"{name}_pred"])


@pytest.mark.parametrize("seed,n,F,md,ml", [(0, 5000, 47, 6, 4), (1, 3000, 20, 9, 1), (2, 700, 3, 30, 2)])
def test_gbdt_matches_oracle_on_random_data(cuda_ok, seed, n, F, md, ml):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n, F))
    X[:, ::3] = np.round(X[:, ::3], 1)  # ties in a third of the columns
    # signed zeros: numpy's stable argsort treats -0.0 == 0.0 (the device presort must too)
    X[:, 1] = rng.choice([-0.0, 0.0, 0.5, -0.5], size=n)
    y = np.tanh(X[:, 0]) + 0.3 * X[:, 1] * X[:, 2 % F] + 0.05 * rng.normal(size=n)
    Xv = rng.normal(size=(257, F))
    m = _fit(X, y, Xv, y[:257], 6, md, 0.2, ml)
    base, trees, curve = ogbdt.fit(X, y, num_trees=6, max_depth=md, learning_rate=0.2, min_samples_leaf=ml,
                                   eval_set=(Xv, y[:257]))
    assert m.base_prediction_ == base
    for got, want in zip(m.trees_, trees):
        for i, k in enumerate(("feature", "threshold", "left", "right", "value")):
            assert np.array_equal(getattr(got, k), want[i]), k
    assert m.train_curve_ == curve
    assert np.array_equal(m.predict(Xv), ogbdt.predict(base, trees, 0.2, Xv))


def test_gbdt_weights_round_trip_and_validation(cuda_ok):
    from paper_2304_05430_b200 import GradientBoostedTrees
    from paper_2304_05430_b200.errors import DataValidationError

    g = golden("gbdt.npz")
    m = _fit(g["conv_X"], g["conv_y"], g["conv_Xv"], g["conv_yv"], 5, 4, 0.1, 4)
    m2 = GradientBoostedTrees(learning_rate=0.1)
    m2.set_weights(m.get_weights())
    assert np.array_equal(m2.predict(g["conv_Xv"]), m.predict(g["conv_Xv"]))
    assert np.array_equal(m.predict(g["conv_Xv"][:7]), m.predict(g["conv_Xv"])[:7])  # cached trees
    assert m2.train_curve_ == []
    with pytest.raises(DataValidationError, match="num_trees"):
        GradientBoostedTrees(num_trees=0).fit(np.zeros((3, 2)), np.zeros(3))
    with pytest.raises(DataValidationError, match="non-finite"):
        GradientBoostedTrees().fit(np.array([[np.nan]]), np.zeros(1))
    with pytest.raises(DataValidationError, match="before fit"):
        GradientBoostedTrees().predict(np.zeros((1, 1)))
    with pytest.raises(DataValidationError, match="expected 47 features"):
        m.predict(np.zeros((2, 3)))
    assert m.predict(np.zeros((0, 47))).shape == (0,)
