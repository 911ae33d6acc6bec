"""Shared test plumbing.

* registers the ``gpu`` marker (tests that need a B200; the driver runs
  ``-m "not gpu"`` on CPU and ``-m gpu`` on the box);
* puts the repo root on sys.path so ``oracle`` (the CPU checker) and the
  product package import from the working tree;
* helpers that load the committed golden fixtures and rebuild the
  duck-typed step sequences the reference's estimators consume.
"""

from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@dataclass
class Seq:
    """Duck-typed StepSequence (features.py:70-92): .steps (T, d0), .context (C,)."""

    steps: np.ndarray
    context: np.ndarray


def golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def unpack_seqs(steps, off, ctx):
    return [Seq(steps[off[i]:off[i + 1]], ctx[i]) for i in range(len(off) - 1)]


def segments(a, b, off):
    return [(a[off[i]:off[i + 1]], b[off[i]:off[i + 1]]) for i in range(len(off) - 1)]


def random_seqs(rng, lengths, d0=6, C=35):
    return [Seq(rng.normal(size=(int(t), d0)), rng.normal(size=C)) for t in lengths]


def central_difference_grads(loss_fn, params: dict, eps: float = 1e-6) -> dict:
    """Same definition as the reference's tests/conftest.py:56-75."""
    out = {}
    for name, arr in params.items():
        g = np.zeros_like(arr, dtype=np.float64)
        flat, gf = arr.reshape(-1), g.reshape(-1)
        for i in range(flat.size):
            keep = flat[i]
            flat[i] = keep + eps
            up = loss_fn()
            flat[i] = keep - eps
            dn = loss_fn()
            flat[i] = keep
            gf[i] = (up - dn) / (2.0 * eps)
        out[name] = g
    return out


def relative_gradient_error(analytic: dict, numeric: dict) -> float:
    """Norm-ratio error with a 1e-4 floor (reference tests/conftest.py:78-96)."""
    worst = 0.0
    for name in numeric:
        a = np.asarray(analytic[name], dtype=np.float64).ravel()
        n = np.asarray(numeric[name], dtype=np.float64).ravel()
        den = max(float(np.linalg.norm(a) + np.linalg.norm(n)), 1e-4)
        worst = max(worst, float(np.linalg.norm(a - n)) / den)
    return worst


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return True
