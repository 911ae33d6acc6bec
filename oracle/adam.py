"""Adam restatement (TEST INFRASTRUCTURE ONLY) <- estimators/optim.py:8-46.

Semantics kept: one shared step counter that advances on every call even
when a parameter is absent from ``grads`` (frozen), bias corrections
1 - beta^t, epsilon added after the square root of the corrected second
moment, parameters updated in place.
"""

from __future__ import annotations

import numpy as np


class AdamOracle:
    def __init__(self, params: dict, lr: float, b1=0.9, b2=0.999, eps=1e-8):
        self.params = params
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps
        self.m = {k: np.zeros_like(v) for k, v in params.items()}
        self.v = {k: np.zeros_like(v) for k, v in params.items()}
        self.t = 0

    def step(self, grads: dict) -> None:
        self.t += 1
        c1 = 1.0 - self.b1**self.t
        c2 = 1.0 - self.b2**self.t
        for name, g in grads.items():
            m, v = self.m[name], self.v[name]
            m *= self.b1
            m += (1.0 - self.b1) * g
            v *= self.b2
            v += (1.0 - self.b2) * g * g
            self.params[name] -= self.lr * (m / c1) / (np.sqrt(v / c2) + self.eps)
