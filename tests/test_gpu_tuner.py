"""Attention tuner kernels (K5 forward, K6/K7/K8 fused train step) vs the
pinned oracle and the reference's golden vectors.

Tolerances (stated, SURVEY.md §8c / BASELINE.md §4):
  fp32 build: scores |d| <= 1e-5 abs; loss rel 1e-5; gradients relative-norm
              error <= 1e-4 per tensor.
  fp64 build: scores rel 1e-10; gradients rel 1e-8; training trajectories
              (2 epochs) rel 1e-8 -- the same kernels instantiated in double.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import (central_difference_grads, golden, random_seqs, relative_gradient_error,
                      unpack_seqs)
from oracle import tuner as otuner

pytestmark = pytest.mark.gpu


def make(precision, **kw):
    from paper_2304_05430_b200 import RecurrentAttentionTuner

    m = RecurrentAttentionTuner(**kw)
    m.precision = precision
    return m


def test_init_is_bit_identical_to_reference(cuda_ok):
    g = golden("tuner.npz")
    seqs = unpack_seqs(g["small_steps"], g["small_off"], g["small_ctx"])
    m = make("fp32", epochs=0, hidden_size=4, recurrent_layers=2, seed=1).fit(seqs, g["small_y"])
    for k, v in m.params_.items():
        assert np.array_equal(v, g["small_init_" + k]), k
    m = make("fp32", epochs=0, seed=0).fit(seqs, g["small_y"])
    names = list(m.params_)
    np.testing.assert_array_equal([m.params_[k].sum() for k in names], g["dflt_init_sum"])


@pytest.mark.parametrize("precision,rtol,atol", [("fp64", 1e-10, 1e-13), ("fp32", 0, 1e-5)])
def test_predict_matches_reference_golden(cuda_ok, precision, rtol, atol):
    g = golden("tuner.npz")
    seqs = unpack_seqs(g["small_steps"], g["small_off"], g["small_ctx"])
    m = make(precision, epochs=0, hidden_size=4, recurrent_layers=2, seed=1).fit(seqs, g["small_y"])
    np.testing.assert_allclose(m.predict(seqs), g["small_pred"], rtol=rtol, atol=atol)
    seqs = unpack_seqs(g["dflt_steps"], g["dflt_off"], g["dflt_ctx"])
    m = make(precision, epochs=0, seed=0).fit(seqs, g["dflt_y"])
    np.testing.assert_allclose(m.predict(seqs), g["dflt_pred"], rtol=rtol, atol=atol)


@pytest.mark.parametrize("precision,rtol,gtol", [("fp64", 1e-10, 1e-8), ("fp32", 1e-5, 1e-4)])
def test_loss_and_gradients_match_reference_golden(cuda_ok, precision, rtol, gtol):
    g = golden("tuner.npz")
    seqs = unpack_seqs(g["small_steps"], g["small_off"], g["small_ctx"])
    for loss in ("rmse", "ranking"):
        m = make(precision, epochs=0, hidden_size=4, recurrent_layers=2, seed=1, loss=loss)
        m.fit(seqs, g["small_y"])
        l, gr = m.loss_and_gradients(seqs, g["small_y"])
        assert l == pytest.approx(float(g[f"small_{loss}_loss"]), rel=rtol)
        want = {k: g[f"small_{loss}_g_{k}"] for k in gr}
        assert relative_gradient_error(gr, want) <= gtol
    seqs = unpack_seqs(g["dflt_steps"], g["dflt_off"], g["dflt_ctx"])
    for loss in ("rmse", "ranking"):
        m = make(precision, epochs=0, seed=0, loss=loss).fit(seqs, g["dflt_y"])
        l, gr = m.loss_and_gradients(seqs[:16], g["dflt_y"][:16])
        assert l == pytest.approx(float(g[f"dflt_{loss}_loss"]), rel=rtol)
        names = list(m.params_)
        np.testing.assert_allclose([np.linalg.norm(gr[k]) for k in names], g[f"dflt_{loss}_gnorm"],
                                   rtol=gtol * 10)
        p = otuner.init_params(0)
        _, og = otuner.loss_and_gradients(p, seqs[:16], g["dflt_y"][:16], loss)
        assert relative_gradient_error(gr, og) <= gtol


def test_predict_padding_and_chunk_invariance(cuda_ok):
    rng = np.random.default_rng(11)
    seqs = random_seqs(rng, (1, 7, 3, 5, 2, 32, 9))
    m = make("fp32", epochs=0, seed=5).fit(seqs, rng.uniform(0.2, 0.8, size=len(seqs)))
    batched = m.predict(seqs)
    singles = np.array([m.predict([s])[0] for s in seqs])
    assert np.array_equal(batched, singles)  # per-program arithmetic is independent of the tile
    assert np.array_equal(m.predict(seqs, chunk=3), batched)
    out = m.predict(seqs * 3)
    assert np.all((out > 0) & (out < 1))
    assert m.predict([]).shape == (0,)


@pytest.mark.parametrize("precision", ["fp32", "fp64", "tf32"])
def test_scores_do_not_depend_on_the_launch_size(cuda_ok, precision):
    """Search-time batching (f2) relies on it: a program's score is the same
    whether it is scored alone, in a small launch (one program per CTA) or in
    a bulk launch (multi-program tiles), bit for bit."""
    rng = np.random.default_rng(12)
    seqs = random_seqs(rng, rng.integers(1, 13, size=9))
    m = make(precision, epochs=0, seed=5).fit(seqs, rng.uniform(0.2, 0.8, size=len(seqs)))
    singles = np.array([m.predict([s])[0] for s in seqs])
    for reps in (2, 40, 400):  # 18 / 360 / 3600 programs
        big = m.predict(seqs * reps)
        for r in range(reps):
            np.testing.assert_array_equal(big[r * 9:(r + 1) * 9], singles)


def test_large_random_batch_matches_oracle(cuda_ok):
    rng = np.random.default_rng(99)
    lens = rng.integers(1, 33, size=777)
    seqs = random_seqs(rng, lens)
    y = rng.uniform(0.1, 0.9, size=len(seqs))
    m = make("fp32", epochs=0, seed=3).fit(seqs, y)
    p = otuner.init_params(3)
    want = otuner.predict(p, seqs)
    np.testing.assert_allclose(m.predict(seqs), want, rtol=0, atol=1e-5)
    m64 = make("fp64", epochs=0, seed=3).fit(seqs, y)
    np.testing.assert_allclose(m64.predict(seqs), want, rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("loss", ["rmse", "ranking"])
def test_training_trajectory_matches_reference_fp64(cuda_ok, loss):
    g = golden("tuner.npz")
    seqs = unpack_seqs(g["fit_steps"], g["fit_off"], g["fit_ctx"])
    y, grp = g["fit_y"], list(g["fit_groups"])
    m = make("fp64", epochs=2, batch_size=4, hidden_size=4, recurrent_layers=1, learning_rate=3e-3,
             loss=loss, seed=9)
    m.fit(seqs, y, eval_set=(seqs, y), eval_groups=grp)
    for k, v in m.params_.items():
        np.testing.assert_allclose(v, g[f"fit_{loss}_{k}"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(np.array(m.train_curve_, dtype=np.float64), g[f"fit_{loss}_curve"],
                               rtol=1e-8)
    head = set(m.param_groups()["head"])
    before = {k: v.copy() for k, v in m.params_.items()}
    m.continue_fit(seqs, y, epochs=2, learning_rate=1e-3, trainable=head)
    for k, v in m.params_.items():
        np.testing.assert_allclose(v, g[f"cont_{loss}_{k}"], rtol=1e-8, atol=1e-12)
        if k not in head:
            assert np.array_equal(v, before[k]), k


def test_training_fp32_tracks_oracle(cuda_ok):
    rng = np.random.default_rng(5)
    seqs = random_seqs(rng, rng.integers(1, 11, size=64))
    y = rng.uniform(0.1, 0.9, size=64)
    m = make("fp32", epochs=3, batch_size=16, loss="ranking", seed=2).fit(seqs, y)
    p = otuner.init_params(2)
    curve = otuner.train(p, seqs, y, epochs=3, lr=1e-3, batch_size=16, seed=2, loss="ranking")
    # Adam normalises updates, so fp32-vs-fp64 noise on near-zero gradient
    # entries is amplified to O(lr) per step; compare trajectories in norm.
    np.testing.assert_allclose([c[0] for c in m.train_curve_], [c[0] for c in curve], rtol=1e-3)
    for k in p:
        err = np.linalg.norm(m.params_[k] - p[k]) / max(np.linalg.norm(p[k]), 1e-12)
        assert err <= 2e-3, (k, err)


def test_same_seed_refit_is_bit_identical(cuda_ok):
    rng = np.random.default_rng(21)
    seqs = random_seqs(rng, rng.integers(1, 6, size=40))
    y = rng.uniform(0.1, 0.9, size=40)
    a = make("fp32", epochs=2, batch_size=8, seed=9).fit(seqs, y)
    b = make("fp32", epochs=2, batch_size=8, seed=9).fit(seqs, y)
    assert a.train_curve_ == b.train_curve_
    for k in a.params_:
        assert np.array_equal(a.params_[k], b.params_[k])


def test_gradients_match_central_differences_fp64(cuda_ok):
    """The reference's own FD check (test_tuner.py:83-120) against the fp64 build."""
    rng = np.random.default_rng(3)
    seqs = random_seqs(rng, (2, 5, 3, 4))
    y = rng.uniform(0.1, 0.9, size=4)
    for loss, layers in (("rmse", 2), ("ranking", 1)):
        m = make("fp64", epochs=0, loss=loss, hidden_size=4, recurrent_layers=layers, seed=1)
        m.fit(seqs, y)
        _, analytic = m.loss_and_gradients(seqs, y)
        numeric = central_difference_grads(lambda: m.loss_and_gradients(seqs, y)[0], m.params_)
        for names in m.param_groups().values():
            err = relative_gradient_error({k: analytic[k] for k in names},
                                          {k: numeric[k] for k in names})
            assert err <= 1e-3


def test_divergence_names_the_epoch(cuda_ok):
    from paper_2304_05430_b200.errors import NumericFailure

    rng = np.random.default_rng(21)
    seqs = random_seqs(rng, rng.integers(1, 6, size=24))
    y = rng.uniform(0.1, 0.9, size=24)
    with pytest.raises(NumericFailure, match="epoch 0"):
        make("fp32", epochs=2, learning_rate=1e200, hidden_size=4, recurrent_layers=1).fit(seqs, y)


def test_validation_matches_reference(cuda_ok):
    from paper_2304_05430_b200.errors import DataValidationError

    rng = np.random.default_rng(0)
    seqs = random_seqs(rng, (2,))
    with pytest.raises(DataValidationError, match="unknown loss"):
        make("fp32", loss="mae").fit(seqs, np.array([0.5]))
    for kw in ({"batch_size": 0}, {"epochs": -1}, {"hidden_size": 0}, {"recurrent_layers": 0},
               {"attention_heads": 0}, {"attention_unroll_steps": 0},
               {"attention_heads": 3, "hidden_size": 8}):
        with pytest.raises(DataValidationError):
            make("fp32", **kw).fit(seqs, np.array([0.5]))
    with pytest.raises(DataValidationError, match="non-empty"):
        make("fp32").fit([], np.zeros(0))
    with pytest.raises(DataValidationError, match="before fit"):
        make("fp32").predict([])
    with pytest.raises(DataValidationError, match="before fit"):
        make("fp32").continue_fit([], np.zeros(0), 1, 1e-3)


def test_weight_round_trip_preserves_predictions(cuda_ok):
    rng = np.random.default_rng(14)
    seqs = random_seqs(rng, rng.integers(1, 6, size=20))
    y = rng.uniform(0.1, 0.9, size=20)
    m = make("fp32", epochs=1, hidden_size=4, recurrent_layers=1, seed=6).fit(seqs, y)
    clone = make("fp32", hidden_size=4, recurrent_layers=1, attention_heads=2)
    clone.set_weights(m.get_weights())
    assert np.array_equal(clone.predict(seqs), m.predict(seqs))


@pytest.mark.parametrize("precision", ["fp32", "fp32_cuda", "tf32", "fp64"])
def test_concurrent_predict_from_worker_threads(cuda_ok, precision):
    """search.tune(jobs>1) calls predict from ThreadPoolExecutor workers
    (search.py:563-567; SPEC.md:538 'safe for concurrent predict'): results
    from 8 threads x mixed batch sizes (and longest programs, i.e. shared-memory
    sizes of the same kernel) equal the serial ones bit for bit."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(7)
    seqs = random_seqs(rng, rng.integers(1, 13, 600))
    m = make(precision, epochs=0, seed=3).fit(seqs, rng.uniform(size=600))
    chunks = [seqs[i:i + n] for i, n in zip(range(0, 600, 37), [1, 5, 32, 37] * 40)]
    serial = [m.predict(c) for c in chunks]
    with ThreadPoolExecutor(max_workers=8) as ex:
        for _ in range(3):
            got = list(ex.map(m.predict, chunks))
            for a, b in zip(got, serial):
                np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("precision,kw,tol", [
    ("fp64", dict(hidden_size=4, recurrent_layers=1), 1e-9),
    ("fp32", dict(), 2e-3),   # latency-path kernel (hidden 32); relative norm per tensor
])
def test_numeric_failure_keeps_state_of_last_finite_step(cuda_ok, precision, kw, tol):
    """after NumericFailure, params_ hold the state as of the last
    finite minibatch, like the reference's in-place Adam (tuner.py:449-450).
    A NaN label placed in minibatch 3 of epoch 0: three Adam steps happen,
    then both the oracle's loop and the kernel stop."""
    from oracle import tuner as otuner
    from paper_2304_05430_b200.errors import NumericFailure

    rng = np.random.default_rng(31)
    seqs = random_seqs(rng, rng.integers(1, 8, size=64))
    y = rng.uniform(0.1, 0.9, size=64)
    y[int(np.random.default_rng(0 + 1).permutation(64)[3 * 8 + 2])] = np.nan
    p = otuner.init_params(0, layers=kw.get("recurrent_layers", 3), hidden=kw.get("hidden_size", 32))
    with pytest.raises(FloatingPointError, match="epoch 0"):
        otuner.train(p, seqs, y, epochs=3, lr=1e-3, batch_size=8, seed=0)
    m = make(precision, epochs=3, batch_size=8, seed=0, **kw)
    with pytest.raises(NumericFailure, match="epoch 0"):
        m.fit(seqs, y)
    init = otuner.init_params(0, layers=kw.get("recurrent_layers", 3), hidden=kw.get("hidden_size", 32))
    assert any(not np.array_equal(p[k], init[k]) for k in p)  # the 3 steps did update
    for k, v in p.items():
        err = np.linalg.norm(m.params_[k] - v) / max(np.linalg.norm(v), 1e-12)
        assert err <= tol, (k, err)
