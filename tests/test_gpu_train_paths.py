"""The two tuner training kernels behind tt_tuner_train_f32:

* the v4 latency path (csrc/tt_tuner_fast.cuh): hidden 32, batch <= #SMs,
  per-sample caches in shared memory, weight gradients reduced by
  parameter-slice jobs;
* the generic kernel (csrc/tt_tuner.cu tuner_train_kernel): any hidden size,
  per-CTA partial gradients.

Both are checked against the float64 oracle (oracle/tuner.py, pinned to the
reference goldens) and against each other.  Tolerances as test_gpu_tuner.py:
fp32 loss rel 1e-5, gradients relative-norm 1e-4 per tensor, trajectories in
norm (Adam amplifies fp32 noise on near-zero gradient entries).
"""

from __future__ import annotations

import contextlib

import numpy as np
import pytest

from conftest import random_seqs, relative_gradient_error
from oracle import tuner as otuner

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def train_path(path: int):
    from paper_2304_05430_b200 import _lib

    _lib.call("tt_tuner_train_set_path", path)
    try:
        yield
    finally:
        _lib.call("tt_tuner_train_set_path", 0)


def make(**kw):
    from paper_2304_05430_b200 import RecurrentAttentionTuner

    m = RecurrentAttentionTuner(**kw)
    m.precision = "fp32"
    return m


def _grads(m, seqs, y):
    loss, g = m.loss_and_gradients(seqs, y)
    return loss, g


@pytest.mark.parametrize("loss", ["rmse", "ranking"])
def test_fast_and_generic_gradients_match_oracle(cuda_ok, loss):
    rng = np.random.default_rng(41)
    seqs = random_seqs(rng, rng.integers(1, 11, size=16))
    y = rng.uniform(0.1, 0.9, size=16)
    m = make(epochs=0, seed=4, loss=loss).fit(seqs, y)
    p = otuner.init_params(4)
    want_l, want = otuner.loss_and_gradients(p, seqs, y, loss)
    out = {}
    for path in (1, 2):
        with train_path(path):
            l, g = _grads(m, seqs, y)
        assert l == pytest.approx(want_l, rel=1e-5), path
        assert relative_gradient_error(g, want) <= 1e-4, path
        out[path] = g
    assert relative_gradient_error(out[2], out[1]) <= 1e-4


def test_fast_path_odd_batches(cuda_ok):
    """Batch sizes that leave most CTAs as gradient jobs, single sample,
    length-1 programs, and the maximum step count the smem plan admits."""
    rng = np.random.default_rng(8)
    p = otuner.init_params(6)
    for lens in ([1], [1, 1, 1], [3, 12, 1, 7, 2], list(rng.integers(1, 13, size=33))):
        seqs = random_seqs(rng, lens)
        y = rng.uniform(0.1, 0.9, size=len(seqs))
        m = make(epochs=0, seed=6, loss="ranking").fit(seqs, y)
        with train_path(2):
            l, g = _grads(m, seqs, y)
        want_l, want = otuner.loss_and_gradients(p, seqs, y, "ranking")
        assert l == pytest.approx(want_l, rel=1e-5, abs=1e-7)
        if want_l > 0:
            assert relative_gradient_error(g, want) <= 1e-4, lens


def test_fast_path_tenset_width(cuda_ok):
    """164-wide step rows (the tuner is width-generic)."""
    rng = np.random.default_rng(2)
    seqs = random_seqs(rng, rng.integers(1, 9, size=12), d0=164)
    y = rng.uniform(0.1, 0.9, size=12)
    p = otuner.init_params(1, d0=164)
    m = make(epochs=0, seed=1, loss="ranking")
    m.set_weights(p)
    np.testing.assert_allclose(m.predict(seqs), otuner.predict(p, seqs), rtol=0, atol=1e-5)
    with train_path(2):
        l, g = _grads(m, seqs, y)
    want_l, want = otuner.loss_and_gradients(p, seqs, y, "ranking")
    assert l == pytest.approx(want_l, rel=1e-5)
    assert relative_gradient_error(g, want) <= 1e-4


@pytest.mark.parametrize("loss", ["rmse", "ranking"])
def test_fast_path_trajectory_with_partial_batch(cuda_ok, loss):
    rng = np.random.default_rng(13)
    seqs = random_seqs(rng, rng.integers(1, 11, size=37))  # 2 x 16 + 5
    y = rng.uniform(0.1, 0.9, size=37)
    with train_path(2):
        m = make(epochs=2, batch_size=16, loss=loss, seed=3).fit(seqs, y)
    p = otuner.init_params(3)
    curve = otuner.train(p, seqs, y, epochs=2, lr=1e-3, batch_size=16, seed=3, loss=loss)
    np.testing.assert_allclose([c[0] for c in m.train_curve_], [c[0] for c in curve], rtol=1e-3)
    for k in p:
        err = np.linalg.norm(m.params_[k] - p[k]) / max(np.linalg.norm(p[k]), 1e-12)
        assert err <= 2e-3, (k, err)


def test_fast_path_frozen_groups_and_refit(cuda_ok):
    rng = np.random.default_rng(17)
    seqs = random_seqs(rng, rng.integers(1, 9, size=48))
    y = rng.uniform(0.1, 0.9, size=48)
    with train_path(2):
        a = make(epochs=1, batch_size=16, loss="ranking", seed=5).fit(seqs, y)
        b = make(epochs=1, batch_size=16, loss="ranking", seed=5).fit(seqs, y)
        for k in a.params_:
            assert np.array_equal(a.params_[k], b.params_[k]), k  # deterministic reduction
        groups = a.param_groups()
        heads = set(groups["attention"]) | set(groups["head"])
        before = {k: v.copy() for k, v in a.params_.items()}
        a.continue_fit(seqs, y, epochs=1, learning_rate=1e-3, trainable=heads)
    changed = 0
    for k, v in a.params_.items():
        if k in heads:
            changed += int(not np.array_equal(v, before[k]))
        else:
            assert np.array_equal(v, before[k]), k
    assert changed > 0


def test_fast_and_generic_epochs_agree(cuda_ok):
    rng = np.random.default_rng(23)
    seqs = random_seqs(rng, rng.integers(1, 11, size=96))
    y = rng.uniform(0.1, 0.9, size=96)
    res = {}
    for path in (1, 2):
        with train_path(path):
            res[path] = make(epochs=2, batch_size=16, loss="ranking", seed=8).fit(seqs, y)
    np.testing.assert_allclose([c[0] for c in res[1].train_curve_],
                               [c[0] for c in res[2].train_curve_], rtol=1e-4)
    for k in res[1].params_:
        a, b = res[1].params_[k], res[2].params_[k]
        assert np.linalg.norm(a - b) <= 1e-3 * max(np.linalg.norm(a), 1e-12), k


@pytest.mark.parametrize("n,loss", [(149, "ranking"), (300, "rmse"), (1024, "ranking")])
def test_multi_round_gradients_match_oracle(cuda_ok, n, loss):
    """Minibatches larger than the grid: several slots per CTA (forward of
    every slot, loss, recomputed forward + backward per slot)."""
    rng = np.random.default_rng(n)
    seqs = random_seqs(rng, rng.integers(1, 11, size=n))
    y = rng.uniform(0.1, 0.9, size=n)
    m = make(epochs=0, seed=2, loss=loss).fit(seqs, y)
    p = otuner.init_params(2)
    want_l, want = otuner.loss_and_gradients(p, seqs, y, loss)
    res = {}
    for path in (1, 2):
        with train_path(path):
            l, g = _grads(m, seqs, y)
        assert l == pytest.approx(want_l, rel=1e-5), path
        assert relative_gradient_error(g, want) <= 1e-4, path
        res[path] = g
    assert relative_gradient_error(res[2], res[1]) <= 1e-4


def test_multi_round_trajectory(cuda_ok):
    rng = np.random.default_rng(31)
    seqs = random_seqs(rng, rng.integers(1, 11, size=700))  # 2 x 300 + 100
    y = rng.uniform(0.1, 0.9, size=700)
    with train_path(2):
        m = make(epochs=2, batch_size=300, loss="ranking", seed=4).fit(seqs, y)
    p = otuner.init_params(4)
    curve = otuner.train(p, seqs, y, epochs=2, lr=1e-3, batch_size=300, seed=4, loss="ranking")
    np.testing.assert_allclose([c[0] for c in m.train_curve_], [c[0] for c in curve], rtol=1e-3)
    for k in p:
        err = np.linalg.norm(m.params_[k] - p[k]) / max(np.linalg.norm(p[k]), 1e-12)
        assert err <= 2e-3, (k, err)


@pytest.mark.parametrize("batch", [16, 200])
def test_heads_only_finetune_matches_oracle(cuda_ok, batch):
    """continue_fit with only the attention + head groups trainable runs the
    heads-only kernel (frozen last-layer LSTM outputs computed once); the
    trajectory follows the oracle's filtered-gradient Adam (tuner.py:397-425)
    and the full-step kernels."""
    rng = np.random.default_rng(batch)
    seqs = random_seqs(rng, rng.integers(1, 11, size=450))
    y = rng.uniform(0.1, 0.9, size=450)
    base = make(epochs=1, batch_size=batch, loss="ranking", seed=5).fit(seqs, y)
    p0 = {k: v.copy() for k, v in base.params_.items()}
    g = base.param_groups()
    heads = set(g["attention"]) | set(g["head"])
    base.continue_fit(seqs, y, epochs=2, learning_rate=1e-3, trainable=heads)
    for k in g["recurrent"]:
        assert np.array_equal(base.params_[k], p0[k]), k
    p = {k: v.copy() for k, v in p0.items()}
    curve = otuner.train(p, seqs, y, epochs=2, lr=1e-3, batch_size=batch, seed=5, seed_offset=9001,
                         trainable=heads, loss="ranking")
    np.testing.assert_allclose([c[0] for c in base.train_curve_], [c[0] for c in curve], rtol=1e-3)
    # fine-tuning from trained weights: the small bias gradients carry fp32
    # noise that Adam's normalisation amplifies, hence the looser norm bound
    for k in heads:
        err = np.linalg.norm(base.params_[k] - p[k]) / max(np.linalg.norm(p[k]), 1e-12)
        assert err <= 1e-2, (k, err)
    # the generic kernel (full steps with the trainable mask) agrees
    full = make(epochs=0, batch_size=batch, loss="ranking", seed=5).fit(seqs[:2], y[:2])
    full.set_weights(p0)
    with train_path(1):
        full.continue_fit(seqs, y, epochs=2, learning_rate=1e-3, trainable=heads)
    np.testing.assert_allclose([c[0] for c in base.train_curve_], [c[0] for c in full.train_curve_],
                               rtol=1e-4)
    for k in heads:
        err = np.linalg.norm(base.params_[k] - full.params_[k]) / max(np.linalg.norm(full.params_[k]), 1e-12)
        assert err <= (1e-3 if batch <= 16 else 1e-2), (k, err)


def test_long_programs_warn_about_the_generic_kernel(cuda_ok):
    """the 2.4-7x slowdown for programs longer than the latency
    path's shared-memory caches was silent; it now says so (and stays exact)."""
    import warnings

    from conftest import random_seqs
    from paper_2304_05430_b200 import RecurrentAttentionTuner
    from paper_2304_05430_b200.estimators import PerformanceWarning

    rng = np.random.default_rng(1)
    short = random_seqs(rng, rng.integers(1, 8, size=24))
    long_ = random_seqs(rng, [30] + list(rng.integers(1, 8, size=23)))
    y = rng.uniform(0.1, 0.9, size=24)
    with warnings.catch_warnings():
        warnings.simplefilter("error", PerformanceWarning)
        RecurrentAttentionTuner(epochs=1, batch_size=8).fit(short, y)
    with pytest.warns(PerformanceWarning, match="generic kernel"):
        RecurrentAttentionTuner(epochs=1, batch_size=8).fit(long_, y)


@pytest.mark.parametrize("precision,hidden,layers", [("fp64", 4, 1), ("fp32", 32, 3)])
def test_training_with_programs_without_steps(cuda_ok, precision, hidden, layers):
    """The reference trains on programs without steps (masked out, context
    kept); so do the kernels -- generic (fp64) and latency path (fp32)."""
    from conftest import Seq, random_seqs
    from oracle import tuner as otuner
    from paper_2304_05430_b200 import RecurrentAttentionTuner

    rng = np.random.default_rng(51)
    seqs = random_seqs(rng, rng.integers(1, 9, size=48))
    for i in (5, 17, 30):
        seqs[i] = Seq(np.zeros((0, 6)), seqs[i].context)
    y = rng.uniform(0.1, 0.9, size=48)
    m = RecurrentAttentionTuner(epochs=2, batch_size=8, hidden_size=hidden, recurrent_layers=layers,
                                loss="ranking", seed=4)
    m.precision = precision
    m.fit(seqs, y)
    p = otuner.init_params(4, layers=layers, hidden=hidden)
    curve = otuner.train(p, seqs, y, epochs=2, lr=1e-3, batch_size=8, seed=4, loss="ranking")
    rt = 1e-8 if precision == "fp64" else 1e-3
    np.testing.assert_allclose([c[0] for c in m.train_curve_], [c[0] for c in curve], rtol=rt)
    for k in p:
        err = np.linalg.norm(m.params_[k] - p[k]) / max(np.linalg.norm(p[k]), 1e-12)
        assert err <= (1e-8 if precision == "fp64" else 2e-3), (k, err)
