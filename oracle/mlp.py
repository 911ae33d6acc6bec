"""CostMLP restated (TEST INFRASTRUCTURE ONLY) <- estimators/mlp.py:38-163.

Architecture F -> 64 -> 64 -> 1, tanh hidden activations, linear output
(mlp.py:72-79); Glorot-uniform init drawn from default_rng(seed) in the
order W1, W2, W3 (mlp.py:59-70); minibatch Adam with a per-epoch
default_rng(seed + 1).permutation (mlp.py:121-143).
"""

from __future__ import annotations

import numpy as np

from .adam import AdamOracle
from .losses import loss_and_dscore

WIDTH = 64
NAMES = ("W1", "b1", "W2", "b2", "W3", "b3")


def glorot(rng: np.random.Generator, fan_in: int, fan_out: int) -> np.ndarray:
    """mlp.py:20-22 -- uniform(-sqrt(6/(in+out)), +sqrt(6/(in+out)))."""
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-lim, lim, size=(fan_in, fan_out))


def init_params(n_features: int, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    p = {}
    p["W1"] = glorot(rng, n_features, WIDTH)
    p["b1"] = np.zeros(WIDTH)
    p["W2"] = glorot(rng, WIDTH, WIDTH)
    p["b2"] = np.zeros(WIDTH)
    p["W3"] = glorot(rng, WIDTH, 1)
    p["b3"] = np.zeros(1)
    return p


def forward(p: dict, X: np.ndarray):
    a1 = np.tanh(X @ p["W1"] + p["b1"])
    a2 = np.tanh(a1 @ p["W2"] + p["b2"])
    return (a2 @ p["W3"] + p["b3"])[:, 0], (X, a1, a2)


def backward(p: dict, saved, d_out: np.ndarray) -> dict:
    X, a1, a2 = saved
    g = {}
    d = d_out[:, None]
    g["W3"] = a2.T @ d
    g["b3"] = d.sum(axis=0)
    d2 = (d @ p["W3"].T) * (1.0 - a2 * a2)
    g["W2"] = a1.T @ d2
    g["b2"] = d2.sum(axis=0)
    d1 = (d2 @ p["W2"].T) * (1.0 - a1 * a1)
    g["W1"] = X.T @ d1
    g["b1"] = d1.sum(axis=0)
    return g


def loss_and_gradients(p: dict, X, y, kind: str):
    out, saved = forward(p, np.asarray(X, dtype=np.float64))
    loss, d = loss_and_dscore(kind, y, out)
    return loss, backward(p, saved, d)


def predict(p: dict, X) -> np.ndarray:
    return forward(p, np.asarray(X, dtype=np.float64))[0]


def fit(X, y, *, batch_size=16, epochs=200, lr=1e-3, loss="rmse", seed=0,
        eval_set=None):
    """Returns (params, curve) exactly as CostMLP.fit leaves them."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    p = init_params(X.shape[1], seed)
    opt = AdamOracle(p, lr)
    rng = np.random.default_rng(seed + 1)
    curve = []
    n = X.shape[0]
    for epoch in range(epochs):
        order = rng.permutation(n)
        for lo in range(0, n, batch_size):
            b = order[lo : lo + batch_size]
            val, g = loss_and_gradients(p, X[b], y[b], loss)
            if not np.isfinite(val):
                raise FloatingPointError(f"loss became non-finite at epoch {epoch}")
            opt.step(g)
        tr = float(np.sqrt(np.mean((predict(p, X) - y) ** 2)))
        va = None
        if eval_set is not None:
            Xv = np.asarray(eval_set[0], dtype=np.float64)
            yv = np.asarray(eval_set[1], dtype=np.float64)
            va = float(np.sqrt(np.mean((predict(p, Xv) - yv) ** 2)))
        curve.append((tr, va))
    return p, curve
