"""Dataset-pruning statistics on the GPU (sampling.py:37-85).

filter_invalid   <- sampling.py:37-59: per task, throughput of the valid
                    records (data.py:440-446), numpy linear quantile, keep
                    t >= threshold, keep the task iff survivors >= min.  The
                    arithmetic runs in the K2 kernel, bit-exact with numpy
                    float64; selection sets are identical to the reference.
filter_stats     array-level entry point (CSR by task) used by the above.
task_weights / task_priority_order / raw_task_weights <- sampling.py:62-85,
                    host code by design: Python integers (flop counts up to
                    2**63 times occurrence) are exact only on the host.

``prune_dataset`` itself (the sequential rng.choice loop, sampling.py:128-200)
stays on the host: ``install()`` swaps ``tensortune.sampling.filter_invalid``
so the reference's own loop runs on top of this kernel.
"""

from __future__ import annotations

import numpy as np

from . import _device, _lib
from .errors import DataValidationError


def filter_stats(flops, cost, valid, task_offsets, q: float, min_records: int):
    """(threshold[t], keep[r], survivors[t], task_keep[t]) for CSR task groups."""
    t = _device.require_cuda()
    off = np.ascontiguousarray(np.asarray(task_offsets, dtype=np.int64))
    n_tasks = off.shape[0] - 1
    n = int(off[-1]) if n_tasks >= 0 else 0
    dfl = _device.to_dev(np.asarray(flops, dtype=np.int64))
    dco = _device.to_dev(np.nan_to_num(np.asarray(cost, dtype=np.float64), nan=1.0))
    dva = _device.to_dev(np.asarray(valid, dtype=np.uint8))
    doff = _device.to_dev(off)
    thr = _device.empty(max(n_tasks, 1), t.float64)
    keep = _device.empty(max(n, 1), t.uint8)
    surv = _device.empty(max(n_tasks, 1), t.int32)
    tkeep = _device.empty(max(n_tasks, 1), t.uint8)
    _lib.call("tt_prune_stats", dfl.data_ptr(), dco.data_ptr(), dva.data_ptr(), doff.data_ptr(),
              n_tasks, float(q), int(min_records), thr.data_ptr(), keep.data_ptr(), surv.data_ptr(),
              tkeep.data_ptr(), None, 0, _device.stream_ptr())
    return (thr.cpu().numpy()[:n_tasks], keep.cpu().numpy()[:n].astype(bool),
            surv.cpu().numpy()[:n_tasks].astype(np.int64), tkeep.cpu().numpy()[:n_tasks].astype(bool))


def _dataset_arrays(ds):
    """Flatten a tensortune Dataset (duck-typed) into CSR-by-task arrays in
    records_by_task order (the order valid_records_of_task uses)."""
    flops, cost, valid, rids, off = [], [], [], [], [0]
    for task in ds.tasks:
        for rid in ds.records_by_task.get(task.task_id, []):
            r = ds.record_by_id[rid]
            ok = not r.error_flag
            if ok and r.mean_cost is None:
                raise DataValidationError(
                    f"record {r.record_id!r}: throughput is undefined for error records")
            flops.append(int(r.measured_flops) if ok else 0)
            cost.append(float(r.mean_cost) if ok else 1.0)
            valid.append(ok)
            rids.append(rid)
        off.append(len(rids))
    return (np.array(flops, dtype=np.int64), np.array(cost, dtype=np.float64),
            np.array(valid, dtype=bool), np.array(off, dtype=np.int64), rids)


def filter_invalid(ds, cfg):
    """Drop error records, per-task low-throughput tails, and sparse tasks."""
    cfg.validate()
    flops, cost, valid, off, rids = _dataset_arrays(ds)
    if len(ds.tasks) and off[-1] > 0:
        _, keep, _, tkeep = filter_stats(flops, cost, valid, off, cfg.low_perf_quantile,
                                         cfg.min_records_per_task)
    else:
        keep = np.zeros(len(rids), dtype=bool)
        tkeep = np.zeros(len(ds.tasks), dtype=bool)
    keep_tasks = {t.task_id for t, k in zip(ds.tasks, tkeep) if k}
    keep_records = {rid for rid, k in zip(rids, keep) if k}
    tasks = [t for t in ds.tasks if t.task_id in keep_tasks]
    records = [r for r in ds.records if r.record_id in keep_records]
    return type(ds).build(list(ds.hardware), tasks, records, validate=False)


def _flop_count(kernel) -> int:
    try:
        from tensortune.workload import flop_count
    except Exception:  # noqa: BLE001 - duck-typed kernels in tests
        return int(kernel.flops)
    return int(flop_count(kernel))


def raw_task_weights(ds) -> dict:
    occurrence: dict = {}
    for task in ds.tasks:
        occurrence[task.kernel.op] = occurrence.get(task.kernel.op, 0) + 1
    return {t.task_id: float(_flop_count(t.kernel) * occurrence[t.kernel.op]) for t in ds.tasks}


def task_weights(ds) -> dict:
    if not ds.tasks:
        raise DataValidationError("task_weights: dataset has no tasks")
    raw = raw_task_weights(ds)
    total = sum(raw.values())
    return {tid: w / total for tid, w in raw.items()}


def task_priority_order(ds, task_ids=None) -> list:
    raw = raw_task_weights(ds)
    pool = list(raw) if task_ids is None else list(task_ids)
    return sorted(pool, key=lambda tid: (-raw[tid], tid))
