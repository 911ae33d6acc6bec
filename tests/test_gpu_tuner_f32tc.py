"""fp32 tuner scoring on the tensor cores (csrc/tt_tuner_x3.cu) vs the float64
oracle, at the fp32 predict tolerance (atol 1e-5).

The biLSTM gate GEMMs run on tcgen05 in split precision (x.w = x_hi.w_hi +
x_lo.w_hi + x_hi.w_lo, tf32 parts, fp32 accumulation), the activations and
the attention + head are fp32 CUDA-core code.  "fp32" routes here whenever
the model's shapes are covered (hidden 32, heads 1/2/4, step width <= 32);
"fp32_cuda" forces the CUDA-core kernel.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import random_seqs
from oracle import tuner as otuner

pytestmark = pytest.mark.gpu

ATOL = 1e-5


def make(precision="fp32", **kw):
    from paper_2304_05430_b200 import RecurrentAttentionTuner

    m = RecurrentAttentionTuner(**kw)
    m.precision = precision
    return m


def test_fp32_routes_to_the_tensor_core_kernel(cuda_ok):
    from paper_2304_05430_b200 import _lib

    rng = np.random.default_rng(1)
    seqs = random_seqs(rng, rng.integers(1, 9, size=50))
    m = make(epochs=0, seed=3).fit(seqs, rng.uniform(0.1, 0.9, size=50))
    before = _lib.CALLS["tt_tuner_predict_f32tc"], _lib.CALLS["tt_tuner_predict_f32"]
    tc = m.predict(seqs)
    assert _lib.CALLS["tt_tuner_predict_f32tc"] == before[0] + 1
    m.precision = "fp32_cuda"
    cu = m.predict(seqs)
    assert _lib.CALLS["tt_tuner_predict_f32"] == before[1] + 1
    np.testing.assert_allclose(tc, cu, rtol=0, atol=ATOL)


@pytest.mark.parametrize("lens_hi,n", [(11, 777), (33, 300), (2, 129), (65, 40)])
def test_scores_match_oracle(cuda_ok, lens_hi, n):
    rng = np.random.default_rng(lens_hi)
    seqs = random_seqs(rng, rng.integers(1, lens_hi, size=n))
    m = make(epochs=0, seed=3).fit(seqs, rng.uniform(0.1, 0.9, size=n))
    np.testing.assert_allclose(m.predict(seqs), otuner.predict(otuner.init_params(3), seqs), rtol=0, atol=ATOL)


@pytest.mark.parametrize("layers,heads,unroll", [(1, 1, 1), (2, 2, 3), (3, 4, 2), (4, 1, 2)])
def test_architecture_variants(cuda_ok, layers, heads, unroll):
    rng = np.random.default_rng(layers * 10 + heads)
    seqs = random_seqs(rng, rng.integers(1, 12, size=260))
    m = make(epochs=0, seed=5, recurrent_layers=layers, attention_heads=heads,
             attention_unroll_steps=unroll).fit(seqs, rng.uniform(0.1, 0.9, size=260))
    p = otuner.init_params(5, layers=layers)
    np.testing.assert_allclose(m.predict(seqs), otuner.predict(p, seqs, heads=heads, unroll=unroll),
                               rtol=0, atol=ATOL)


@pytest.mark.parametrize("d0,C", [(1, 0), (17, 3), (32, 64)])
def test_step_and_context_widths(cuda_ok, d0, C):
    """Weights of other step / context widths (set_weights; the layout follows them)."""
    rng = np.random.default_rng(d0 + C)
    m = make(epochs=0, seed=4).fit(*_tiny(rng))
    p = otuner.init_params(4, d0=d0, ctx_len=C)
    m.set_weights(p)
    seqs = random_seqs(rng, rng.integers(1, 10, size=150), d0=d0, C=C)
    np.testing.assert_allclose(m.predict(seqs), otuner.predict(p, seqs), rtol=0, atol=ATOL)


def _tiny(rng):
    seqs = random_seqs(rng, [2, 3])
    return seqs, rng.uniform(0.2, 0.8, size=2)


def test_trained_weights(cuda_ok):
    """Weights moved away from the init (larger, less uniform magnitudes)."""
    rng = np.random.default_rng(7)
    seqs = random_seqs(rng, rng.integers(1, 11, size=512))
    m = make(epochs=3, batch_size=16, loss="ranking", seed=1).fit(seqs, rng.uniform(0.1, 0.9, size=512))
    want = otuner.predict({k: v.copy() for k, v in m.params_.items()}, seqs)
    np.testing.assert_allclose(m.predict(seqs), want, rtol=0, atol=ATOL)


def test_scores_do_not_depend_on_the_launch_or_chunk(cuda_ok):
    """Bit-identical scores alone, in one tile, across tiles and across the
    launch chunks of a bulk call (> 4 tiles per SM = 75,776 programs)."""
    from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms

    rng = np.random.default_rng(12)
    seqs = random_seqs(rng, rng.integers(1, 13, size=9))
    m = make(epochs=0, seed=5).fit(seqs, rng.uniform(0.2, 0.8, size=9))
    singles = np.array([m.predict([s])[0] for s in seqs])
    big = m.predict(seqs * 40)
    for r in range(40):
        np.testing.assert_array_equal(big[r * 9:(r + 1) * 9], singles)
    # 90,000 programs through the device API (two launch chunks)
    reps = 10_000
    steps = np.concatenate([s.steps for s in seqs] * reps)
    lens = np.array([len(s.steps) for s in seqs] * reps)
    off = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    ctx = np.stack([s.context for s in seqs] * reps)
    prog = DevicePrograms(HostPrograms(steps, off, ctx), "fp32")
    out = m.predict_device(prog).cpu().numpy().astype(np.float64)
    np.testing.assert_array_equal(out.reshape(reps, 9), np.broadcast_to(singles, (reps, 9)))


def test_long_programs(cuda_ok):
    """Tmax in the hundreds: the launch chunk shrinks to keep the workspace bounded."""
    rng = np.random.default_rng(21)
    seqs = random_seqs(rng, [300, 1, 17, 250])
    m = make(epochs=0, seed=6).fit(seqs, rng.uniform(0.2, 0.8, size=4))
    np.testing.assert_allclose(m.predict(seqs), otuner.predict(otuner.init_params(6), seqs), rtol=0, atol=ATOL)


def test_uncovered_shapes_use_the_cuda_core_kernel(cuda_ok):
    """hidden != 32 (or heads = 8) scores on the CUDA-core fp32 kernel, at the same tolerance."""
    from paper_2304_05430_b200 import _lib

    rng = np.random.default_rng(31)
    seqs = random_seqs(rng, rng.integers(1, 8, size=60))
    for kw, p in (({"hidden_size": 8}, otuner.init_params(2, hidden=8)), ({"attention_heads": 8}, None)):
        m = make(epochs=0, seed=2, **kw).fit(seqs, rng.uniform(0.1, 0.9, size=60))
        before = _lib.CALLS["tt_tuner_predict_f32"], _lib.CALLS["tt_tuner_predict_f32tc"]
        got = m.predict(seqs)
        assert _lib.CALLS["tt_tuner_predict_f32"] == before[0] + 1
        assert _lib.CALLS["tt_tuner_predict_f32tc"] == before[1]
        want = otuner.predict(p if p is not None else {k: v.copy() for k, v in m.params_.items()}, seqs,
                              heads=kw.get("attention_heads", 2))
        np.testing.assert_allclose(got, want, rtol=0, atol=ATOL)


@pytest.mark.parametrize("precision,atol", [("fp32", ATOL), ("fp32_cuda", ATOL), ("fp64", 1e-12), ("tf32", 2e-3)])
def test_empty_programs(cuda_ok, precision, atol):
    """A program with no steps scores like the reference (pooled and context
    vectors zero), alone and inside a batch; an all-empty batch too."""
    from conftest import Seq

    rng = np.random.default_rng(41)
    seqs = random_seqs(rng, [3, 1, 5])
    m = make(precision, epochs=0, seed=7).fit(seqs, rng.uniform(0.2, 0.8, size=3))
    empty = Seq(np.zeros((0, 6)), rng.normal(size=35))
    batch = [seqs[0], empty, seqs[1], empty, seqs[2]]
    p = otuner.init_params(7)
    got = m.predict(batch)
    np.testing.assert_allclose(got, otuner.predict(p, batch), rtol=0, atol=atol)
    # an all-empty batch (the reference's numpy reshape raises on it): the same scores
    np.testing.assert_array_equal(m.predict([empty, empty]), [got[1], got[3]])
    # whole tiles of empty programs (the reference's 256-program chunks would
    # hit the same reshape): each scores as above, the others as alone
    many = m.predict([empty] * 300 + seqs)
    np.testing.assert_array_equal(many[:300], np.full(300, got[1]))
    np.testing.assert_allclose(many[300:], otuner.predict(p, seqs), rtol=0, atol=atol)


def test_saturated_activations(cuda_ok):
    """Step values large enough to saturate every gate (the cell clamps its
    exponent arguments at +-43 so the shared reciprocals stay finite): still
    within the fp32 tolerance of the float64 oracle, no NaN."""
    rng = np.random.default_rng(61)
    seqs = random_seqs(rng, rng.integers(1, 11, size=200))
    for s in seqs[::2]:
        s.steps *= 300.0  # pre-activations in the hundreds
    m = make(epochs=0, seed=8).fit(seqs, rng.uniform(0.1, 0.9, size=200))
    got = m.predict(seqs)
    assert np.all(np.isfinite(got))
    np.testing.assert_allclose(got, otuner.predict(otuner.init_params(8), seqs), rtol=0, atol=ATOL)
