"""Loss restatements (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

pairwise_logistic  <- estimators/mlp.py:25-35 (ranking_grad)
squared_error      <- estimators/tuner.py:372-375, estimators/mlp.py:105-108
"""

from __future__ import annotations

import numpy as np


def pairwise_logistic(y: np.ndarray, s: np.ndarray) -> tuple[float, np.ndarray]:
    """Mean softplus(-(s_i - s_j)) over ordered pairs y_i > y_j, and d/ds.

    Pair set and normalisation follow mlp.py:27-34: only strictly ordered
    label pairs count (ties contribute nothing), the loss is the mean over
    those pairs, and the gradient for score k is
    (sum_i sigma_ik - sum_j sigma_kj) / n_pairs with sigma = 1/(1+e^margin).
    No ordered pair -> (0.0, zeros)  (mlp.py:29-30).
    """
    y = np.asarray(y, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    above = np.greater.outer(y, y)  # above[i, j] <=> y_i > y_j
    count = int(np.count_nonzero(above))
    if count == 0:
        return 0.0, np.zeros_like(s)
    diff = np.subtract.outer(s, s)  # diff[i, j] = s_i - s_j
    loss = float(np.logaddexp(0.0, -diff[above]).mean())
    weight = np.zeros_like(diff)
    weight[above] = 1.0 / (1.0 + np.exp(diff[above]))
    grad = (weight.sum(axis=0) - weight.sum(axis=1)) / count
    return loss, grad


def squared_error(y: np.ndarray, s: np.ndarray) -> tuple[float, np.ndarray]:
    """mean((s - y)^2) and its gradient 2 (s - y) / B (tuner.py:373-375)."""
    y = np.asarray(y, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    r = s - y
    return float(np.mean(r**2)), 2.0 * r / y.shape[0]


def loss_and_dscore(kind: str, y, s):
    if kind == "ranking":
        return pairwise_logistic(y, s)
    return squared_error(y, s)
