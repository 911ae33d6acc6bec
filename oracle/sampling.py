"""Pruning statistics restated on flat arrays (TEST INFRASTRUCTURE ONLY).

throughput             <- data.py:440-446 (measured_flops / mean_cost)
linear_quantile        <- numpy 2.3.5 np.quantile(method="linear"):
                          virtual index (n-1)*q, floor/next neighbours,
                          clamp at the top, _lerp with the t >= 0.5 branch
                          (numpy/lib/_function_base_impl.py _quantile,
                          _get_indexes, _lerp)
filter_stats           <- sampling.py:37-59 (per-task cut t >= threshold,
                          keep the task iff survivors >= min_records)
raw_task_weights       <- sampling.py:62-69
"""

from __future__ import annotations

import numpy as np


def throughput(flops: np.ndarray, cost: np.ndarray) -> np.ndarray:
    # Python's int / float promotes the int to the nearest double, then
    # performs one IEEE division -- identical to float64 array division.
    return np.asarray(flops, dtype=np.int64).astype(np.float64) / np.asarray(
        cost, dtype=np.float64
    )


def linear_quantile(values: np.ndarray, q: float) -> float:
    """Scalar restatement of np.quantile(values, q) for the linear method."""
    v = np.sort(np.asarray(values, dtype=np.float64))
    n = v.shape[0]
    vi = (n - 1) * float(q)
    if vi >= n - 1:
        return float(v[-1])
    if vi < 0:
        return float(v[0])
    lo = int(np.floor(vi))
    t = vi - lo
    a, b = v[lo], v[lo + 1]
    d = b - a
    if t >= 0.5:
        return float(b - d * (1.0 - t))
    return float(a + d * t)


def filter_stats(flops, cost, valid, task_offsets, q: float, min_records: int):
    """Per-task threshold, record keep mask, survivor counts, task keep flags.

    Records are grouped by task in CSR form (task_offsets, len n_tasks+1);
    ``valid`` marks non-error records.  Tasks with no valid record report a
    NaN threshold, zero survivors and keep=False (sampling.py:49-50).
    """
    flops = np.asarray(flops, dtype=np.int64)
    cost = np.asarray(cost, dtype=np.float64)
    valid = np.asarray(valid, dtype=bool)
    off = np.asarray(task_offsets, dtype=np.int64)
    n_tasks = off.shape[0] - 1
    thr = np.full(n_tasks, np.nan)
    keep = np.zeros(flops.shape[0], dtype=bool)
    surv = np.zeros(n_tasks, dtype=np.int64)
    tkeep = np.zeros(n_tasks, dtype=bool)
    for t in range(n_tasks):
        idx = np.arange(off[t], off[t + 1])
        idx = idx[valid[idx]]
        if idx.size == 0:
            continue
        tp = throughput(flops[idx], cost[idx])
        th = linear_quantile(tp, q)
        thr[t] = th
        ok = tp >= th
        surv[t] = int(ok.sum())
        if surv[t] >= min_records:
            tkeep[t] = True
            keep[idx[ok]] = True
    return thr, keep, surv, tkeep


def raw_task_weights(flop_counts, ops) -> list[float]:
    """float(flop_count * occurrence(op)) per task (sampling.py:62-69)."""
    occ: dict = {}
    for op in ops:
        occ[op] = occ.get(op, 0) + 1
    return [float(int(f) * occ[op]) for f, op in zip(flop_counts, ops)]
