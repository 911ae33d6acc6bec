"""Ranking metrics restated (TEST INFRASTRUCTURE ONLY).

pca_counts / pca       <- metrics.py:46-58 (pairwise_comparison_accuracy)
brute_force_pca        <- tests/conftest.py:26-53 (definition-level loop)
top_k                  <- metrics.py:61-75
rmse                   <- metrics.py:78-81
grouped_pca            <- estimators/tuner.py:486-496, transfer.py:281-290
"""

from __future__ import annotations

import numpy as np


def pca_counts(y, s) -> tuple[int, int]:
    """(#pairs i<j whose label order sign equals the score order sign, #pairs).

    A tie agrees only with a tie (metrics.py:49-51).  Exact integers; the
    reference's float64 mean equals correct/total.
    """
    y = np.asarray(y, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    n = y.shape[0]
    iu = np.triu_indices(n, k=1)
    ly = np.sign(y[iu[0]] - y[iu[1]])
    ls = np.sign(s[iu[0]] - s[iu[1]])
    return int(np.count_nonzero(ly == ls)), int(iu[0].shape[0])


def pca(y, s) -> float:
    c, t = pca_counts(y, s)
    return float(c) / float(t)


def brute_force_pca(y, s) -> float:
    n = len(y)
    good = 0
    tot = 0
    for i in range(n):
        for j in range(i + 1, n):
            a = int(y[i] > y[j]) - int(y[i] < y[j])
            b = int(s[i] > s[j]) - int(s[i] < s[j])
            good += a == b
            tot += 1
    return good / tot


def top_k(y, s, k: int) -> float:
    """max label among the k best-scored entries (stable on ties) / max label."""
    y = np.asarray(y, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    order = np.argsort(-s, kind="stable")
    return float(y[order[:k]].max()) / float(y.max())


def top_k_parts(y, s, k: int) -> tuple[float, float]:
    """(max label over the top-k picks, max label) -- the two kernel outputs."""
    y = np.asarray(y, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    order = np.argsort(-s, kind="stable")
    return float(y[order[:k]].max()), float(y.max())


def rmse(y, s) -> float:
    y = np.asarray(y, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    return float(np.sqrt(np.mean((y - s) ** 2)))


def grouped_pca(y, s, groups) -> float | None:
    """Mean PCA over groups (first-appearance order), singletons skipped."""
    y = np.asarray(y, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    members: dict = {}
    for i, g in enumerate(groups):
        members.setdefault(g, []).append(i)
    vals = [pca(y[ix], s[ix]) for ix in members.values() if len(ix) >= 2]
    return float(np.mean(vals)) if vals else None
