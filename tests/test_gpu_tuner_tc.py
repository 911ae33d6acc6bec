"""Tensor-core (tcgen05, kind::tf32) tuner scoring vs the float64 oracle.

The "tf32" precision mode multiplies tf32-rounded operands (10-bit mantissa)
and accumulates in fp32; the LSTM gates use the hardware tanh (MUFU.TANH,
sigmoid = 0.5 tanh(x/2) + 0.5); softmax and the cell state stay fp32.
Stated tolerance (reduced-precision GEMM operands with fp32
score output): max |d| <= 2e-3 and mean |d| <= 2e-4 against the float64
reference; pairwise order of clearly separated scores is preserved.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import random_seqs
from oracle import tuner as otuner

pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 2e-3, 2e-4


def make(**kw):
    from paper_2304_05430_b200 import RecurrentAttentionTuner

    m = RecurrentAttentionTuner(**kw)
    m.precision = "tf32"
    return m


def _check(got, want):
    d = np.abs(got - want)
    assert d.max() <= MAX_ABS, d.max()
    assert d.mean() <= MEAN_ABS, d.mean()
    assert np.all((got > 0) & (got < 1))


@pytest.mark.parametrize("lens_hi,n", [(11, 777), (33, 300), (2, 129)])
def test_tf32_scores_match_oracle(cuda_ok, lens_hi, n):
    rng = np.random.default_rng(lens_hi)
    seqs = random_seqs(rng, rng.integers(1, lens_hi, size=n))
    y = rng.uniform(0.1, 0.9, size=n)
    m = make(epochs=0, seed=3).fit(seqs, y)
    _check(m.predict(seqs), otuner.predict(otuner.init_params(3), seqs))


@pytest.mark.parametrize("layers,heads,unroll", [(1, 1, 1), (2, 2, 3), (3, 1, 2)])
def test_tf32_architecture_variants(cuda_ok, layers, heads, unroll):
    rng = np.random.default_rng(layers * 10 + heads)
    seqs = random_seqs(rng, rng.integers(1, 12, size=260))
    y = rng.uniform(0.1, 0.9, size=260)
    m = make(epochs=0, seed=5, recurrent_layers=layers, attention_heads=heads,
             attention_unroll_steps=unroll).fit(seqs, y)
    p = otuner.init_params(5, layers=layers)
    _check(m.predict(seqs), otuner.predict(p, seqs, heads=heads, unroll=unroll))


def test_tf32_trained_weights_and_fp32_agreement(cuda_ok):
    """After a few epochs (weights away from init), tf32 scores track both the
    fp32 CUDA-core kernel and the oracle, and preserve clearly separated orders."""
    rng = np.random.default_rng(7)
    seqs = random_seqs(rng, rng.integers(1, 11, size=512))
    y = rng.uniform(0.1, 0.9, size=512)
    m = make(epochs=2, batch_size=16, loss="ranking", seed=1)
    m.precision = "fp32"
    m.fit(seqs, y)
    ref = otuner.predict({k: v.copy() for k, v in m.params_.items()}, seqs)
    fp32 = m.predict(seqs)
    m.precision = "tf32"
    tf = m.predict(seqs)
    _check(tf, ref)
    assert np.abs(tf - fp32).max() <= MAX_ABS
    i, j = np.triu_indices(len(ref), 1)
    sep = np.abs(ref[i] - ref[j]) > 2 * MAX_ABS
    assert np.all(np.sign(tf[i] - tf[j])[sep] == np.sign(ref[i] - ref[j])[sep])


def test_tf32_unsupported_shapes_fall_back(cuda_ok):
    """hidden != 32 routes to the fp32 kernel (no silent wrong answers)."""
    rng = np.random.default_rng(9)
    seqs = random_seqs(rng, rng.integers(1, 6, size=40))
    y = rng.uniform(0.1, 0.9, size=40)
    m = make(epochs=0, seed=2, hidden_size=8).fit(seqs, y)
    p = otuner.init_params(2, hidden=8)
    np.testing.assert_allclose(m.predict(seqs), otuner.predict(p, seqs), rtol=0, atol=1e-5)
