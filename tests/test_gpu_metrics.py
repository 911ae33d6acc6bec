"""K1 PCA counter, K10 top-k and K7 rank loss on the GPU vs the pinned oracle.

Bar: bit-exact for PCA values / counts and top-k; ranking loss within the
float64 build's rounding (rel 1e-12).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, segments
from oracle import losses as oloss
from oracle import metrics as om

pytestmark = pytest.mark.gpu


def test_pca_golden_cases_bit_exact(cuda_ok):
    from paper_2304_05430_b200 import metrics as gm

    g = golden("pca.npz")
    vals = gm.segmented_pca(g["y"], g["s"], g["offsets"])
    np.testing.assert_array_equal(vals, g["pca"])
    # the single-task public API, reference signature
    for (y, s), want in list(zip(segments(g["y"], g["s"], g["offsets"]), g["pca"]))[:40]:
        assert gm.pairwise_comparison_accuracy(y, s) == want


@pytest.mark.parametrize("n", [2, 3, 31, 1023, 1024, 1025, 2048, 4096, 5000, 9000])
def test_pca_counts_match_oracle_across_tile_edges(cuda_ok, n):
    from paper_2304_05430_b200 import metrics as gm

    rng = np.random.default_rng(n)
    y = np.round(rng.normal(size=n), 2)
    s = rng.normal(size=n)
    s[rng.random(n) < 0.2] = 0.0
    s[rng.random(n) < 0.1] = -0.0
    c = gm.pca_counts(y, s, np.array([0, n]))
    want, tot = om.pca_counts(y, s)
    assert int(c[0]) == want


def test_pca_many_ragged_tasks(cuda_ok):
    from paper_2304_05430_b200 import metrics as gm

    rng = np.random.default_rng(11)
    sizes = rng.integers(0, 600, size=150)
    sizes[::17] = 1
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    off[1:] = np.cumsum(sizes)
    y = np.round(rng.normal(size=off[-1]), 1)
    s = np.round(rng.normal(size=off[-1]), 1)
    c = gm.pca_counts(y, s, off)
    for t in range(len(sizes)):
        if sizes[t] >= 2:
            assert int(c[t]) == om.pca_counts(y[off[t]:off[t + 1]], s[off[t]:off[t + 1]])[0]
        else:
            assert int(c[t]) == 0


def test_pca_validation_errors(cuda_ok):
    from paper_2304_05430_b200 import metrics as gm
    from paper_2304_05430_b200.errors import DataValidationError

    with pytest.raises(DataValidationError):
        gm.pairwise_comparison_accuracy([1.0], [1.0])
    with pytest.raises(DataValidationError):
        gm.pairwise_comparison_accuracy([1.0, float("nan")], [1.0, 2.0])
    with pytest.raises(DataValidationError):
        gm.pairwise_comparison_accuracy([1.0, 2.0], [1.0, 2.0, 3.0])


def test_grouped_pca_matches_oracle(cuda_ok):
    from paper_2304_05430_b200 import metrics as gm

    rng = np.random.default_rng(4)
    groups = list(rng.integers(0, 9, size=300))
    y = rng.normal(size=300)
    s = np.round(rng.normal(size=300), 1)
    assert gm.grouped_pca(y, s, groups) == om.grouped_pca(y, s, groups)
    assert gm.grouped_pca(y[:3], s[:3], ["a", "b", "c"]) is None


def test_topk_golden_bit_exact(cuda_ok):
    from paper_2304_05430_b200 import metrics as gm

    g = golden("topk.npz")
    off = g["offsets"]
    for k, key in ((1, "top1"), (5, "top5")):
        pick, best = gm.segmented_topk(g["y"], g["s"], off, k)
        np.testing.assert_array_equal(pick / best, g[key])
    for (y, s), t1 in list(zip(segments(g["y"], g["s"], off), g["top1"]))[:20]:
        assert gm.top_k_score(y, s, 1) == t1


def test_rank_loss_golden(cuda_ok):
    from paper_2304_05430_b200 import metrics as gm

    g = golden("ranking.npz")
    loss, grad = gm.ranking_grad_segments(g["y"], g["s"], g["offsets"], "fp64")
    np.testing.assert_allclose(loss, g["loss"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(grad, g["grad"], rtol=1e-10, atol=1e-15)
    loss32, grad32 = gm.ranking_grad_segments(g["y"], g["s"], g["offsets"], "fp32")
    np.testing.assert_allclose(loss32, g["loss"], rtol=2e-5, atol=1e-6)
    np.testing.assert_allclose(grad32, g["grad"], rtol=1e-4, atol=1e-6)
    for (y, s), want in zip(segments(g["y"], g["s"], g["offsets"]), g["loss"]):
        l, d = oloss.pairwise_logistic(y, s)
        assert l == pytest.approx(want, rel=1e-13)


def test_grouped_pca_rejects_non_finite_scores_like_the_reference(cuda_ok):
    """NaN in a group of >= 2 raises DataValidationError (the
    reference's pairwise_comparison_accuracy -> _as_pair); a NaN in a singleton
    group is never validated by the reference either."""
    from paper_2304_05430_b200 import grouped_pca
    from paper_2304_05430_b200.errors import DataValidationError

    y = np.array([0.1, 0.2, 0.3, 0.4, 0.5])
    s = np.array([0.1, np.nan, 0.3, 0.2, np.inf])
    with pytest.raises(DataValidationError, match="finite"):
        grouped_pca(y, s, ["a", "a", "b", "b", "c"])
    assert grouped_pca(y, s, ["c", "d", "b", "b", "e"]) == 0.0
