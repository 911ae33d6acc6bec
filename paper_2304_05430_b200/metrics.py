"""Ranking metrics on the GPU, with the reference's names and validation.

pairwise_comparison_accuracy  <- metrics.py:46-58   (K1, exact integer counts)
top_k_score                   <- metrics.py:61-75   (K10)
ranking_loss                  <- metrics.py:84-94   (K7 kernel, float64 build)
rmse                          <- metrics.py:78-81   (host; O(n) bookkeeping)
grouped_pca                   <- estimators/tuner.py:486-496 (one K1 launch
                                 for all groups instead of a Python loop)

PCA values are float(correct) / float(total) from exact int64 counts, which
equals the reference's float64 mean of the agreement mask bit for bit.
"""

from __future__ import annotations

import numpy as np

from . import _device, _lib
from .errors import DataValidationError


def _as_pair(y, y_hat, min_n: int):
    """metrics.py:16-29 validation (same messages)."""
    y = np.asarray(y, dtype=np.float64)
    y_hat = np.asarray(y_hat, dtype=np.float64)
    if y.ndim != 1 or y_hat.ndim != 1:
        raise DataValidationError("labels and predictions must be 1-d")
    if y.shape != y_hat.shape:
        raise DataValidationError(
            f"length mismatch: {y.shape[0]} labels vs {y_hat.shape[0]} predictions")
    if y.shape[0] < min_n:
        raise DataValidationError(f"need at least {min_n} entries, got {y.shape[0]}")
    if not (np.isfinite(y).all() and np.isfinite(y_hat).all()):
        raise DataValidationError("labels and predictions must be finite")
    return y, y_hat


def pca_counts(y, y_hat, offsets) -> np.ndarray:
    """Exact concordant-or-jointly-tied pair counts per CSR segment (int64).

    ``y``/``y_hat`` are float64 numpy arrays or CUDA tensors; ``offsets`` is a
    host int64 array of n_segments + 1 entries.
    """
    t = _device.require_cuda()
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    n_tasks = off.shape[0] - 1
    if n_tasks <= 0:
        return np.zeros(0, dtype=np.int64)
    dy = _device.to_dev(y, t.float64)
    ds = _device.to_dev(y_hat, t.float64)
    lib = _lib.load()
    offp = off.ctypes.data_as(_lib.ctypes.c_void_p)
    nbytes = lib.tt_pca_workspace_bytes(offp, n_tasks)
    ws = _device.workspace(nbytes, "pca")
    out = _device.empty(n_tasks, t.int64)
    _lib.call("tt_pca_counts", dy.data_ptr(), ds.data_ptr(), offp, n_tasks, out.data_ptr(),
              ws.data_ptr(), nbytes, _device.stream_ptr())
    return out.cpu().numpy()


def pca_from_counts(counts, offsets) -> np.ndarray:
    n = np.diff(np.asarray(offsets, dtype=np.int64))
    tot = n * (n - 1) // 2
    out = np.full(n.shape, np.nan)
    ok = tot > 0
    out[ok] = counts[ok].astype(np.float64) / tot[ok].astype(np.float64)
    return out


def pairwise_comparison_accuracy(y, y_hat) -> float:
    y, y_hat = _as_pair(y, y_hat, min_n=2)
    c = pca_counts(y, y_hat, np.array([0, y.shape[0]], dtype=np.int64))
    n = y.shape[0]
    return float(int(c[0])) / float(n * (n - 1) // 2)


def segmented_pca(y, y_hat, offsets) -> np.ndarray:
    """Per-segment PCA (NaN for segments with < 2 entries), one launch."""
    return pca_from_counts(pca_counts(y, y_hat, offsets), offsets)


def group_offsets(groups) -> tuple[np.ndarray, np.ndarray]:
    """(permutation, offsets) grouping indices by key in first-appearance order."""
    keys: dict = {}
    for i, g in enumerate(groups):
        keys.setdefault(g, []).append(i)
    perm = np.fromiter((i for idx in keys.values() for i in idx), dtype=np.int64,
                       count=sum(len(v) for v in keys.values()))
    off = np.zeros(len(keys) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(v) for v in keys.values()])
    return perm, off


def grouped_pca(y, y_hat, groups) -> float | None:
    """tuner.py:486-496: mean PCA over groups with >= 2 members, or None."""
    y = np.asarray(y, dtype=np.float64)
    y_hat = np.asarray(y_hat, dtype=np.float64)
    perm, off = group_offsets(groups)
    sizes = np.diff(off)
    if not np.any(sizes >= 2):
        return None
    # the reference validates every group of >= 2 members through
    # pairwise_comparison_accuracy (_as_pair): a NaN score there raises
    # DataValidationError instead of entering the rank sort
    ranked = np.repeat(sizes >= 2, sizes)
    _as_pair(y[perm][ranked], y_hat[perm][ranked], min_n=0)
    vals = segmented_pca(y[perm], y_hat[perm], off)
    scores = [float(v) for v, s in zip(vals, sizes) if s >= 2]
    return float(np.mean(scores))


def segmented_topk(y, y_hat, offsets, k: int) -> tuple[np.ndarray, np.ndarray]:
    """(max label over each segment's min(k, n) best scores, max label)."""
    t = _device.require_cuda()
    off = np.asarray(offsets, dtype=np.int64)
    n_tasks = off.shape[0] - 1
    dy = _device.to_dev(y, t.float64)
    ds = _device.to_dev(y_hat, t.float64)
    doff = _device.to_dev(off)
    pick = _device.empty(n_tasks, t.float64)
    best = _device.empty(n_tasks, t.float64)
    _lib.call("tt_topk", dy.data_ptr(), ds.data_ptr(), doff.data_ptr(), n_tasks, int(k),
              pick.data_ptr(), best.data_ptr(), _device.stream_ptr())
    return pick.cpu().numpy(), best.cpu().numpy()


def top_k_score(y, y_hat, k: int) -> float:
    y, y_hat = _as_pair(y, y_hat, min_n=1)
    n = y.shape[0]
    if not 1 <= k <= n:
        raise DataValidationError(f"k must satisfy 1 <= k <= {n}, got {k}")
    best = float(y.max())
    if best <= 0:
        raise DataValidationError("top_k_score needs a positive best label")
    pick, _ = segmented_topk(y, y_hat, np.array([0, n]), k)
    return float(pick[0]) / best


def rmse(y, y_hat) -> float:
    y, y_hat = _as_pair(y, y_hat, min_n=1)
    return float(np.sqrt(np.mean((y - y_hat) ** 2)))


def ranking_grad_segments(y, s, offsets, precision="fp64"):
    """Pairwise logistic loss and d/ds per segment (K7)."""
    t = _device.require_cuda()
    dt = _device.real_dtype(precision)
    off = np.asarray(offsets, dtype=np.int64)
    n_seg = off.shape[0] - 1
    dy = _device.to_dev(np.asarray(y, dtype=np.float64), dt)
    dsc = _device.to_dev(np.asarray(s, dtype=np.float64), dt)
    doff = _device.to_dev(off)
    loss = _device.empty(n_seg, dt)
    grad = _device.empty(dy.numel(), dt)
    fn = "tt_rank_loss_f64" if precision == "fp64" else "tt_rank_loss_f32"
    max_seg = int(np.max(np.diff(off))) if n_seg else 0
    _lib.call(fn, dy.data_ptr(), dsc.data_ptr(), doff.data_ptr(), n_seg, max_seg, loss.data_ptr(),
              grad.data_ptr(), _device.stream_ptr())
    return loss.cpu().double().numpy(), grad.cpu().double().numpy()


def ranking_grad(y, y_hat):
    """estimators/mlp.py:25-35 on the GPU (float64 build)."""
    y = np.asarray(y, dtype=np.float64)
    y_hat = np.asarray(y_hat, dtype=np.float64)
    if y.shape[0] == 0:
        return 0.0, np.zeros_like(y_hat)
    l, g = ranking_grad_segments(y, y_hat, np.array([0, y.shape[0]]))
    return float(l[0]), g


def ranking_loss(y, y_hat) -> float:
    y, y_hat = _as_pair(y, y_hat, min_n=1)
    return ranking_grad(y, y_hat)[0]
