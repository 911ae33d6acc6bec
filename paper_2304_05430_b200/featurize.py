"""Batched host featurization and labels.

The reference encodes one record at a time and labels each record by
rescanning its task (``features.label``, features.py:199-213: a list of every
valid cost of the task per record, O(n²) per task -- 1,294 records/s at 4096
records per task).  The batch encoders here produce the same arrays, the same
``StepSequence`` objects and the same errors, in one pass:

* labels: the minimum valid cost of each task is computed once per task
  (features.py:206-212: ``min(costs ∪ {c}) / c``);
* context rows (features.py:134-140) are computed once per task and copied
  per record; the flat vector (features.py:103-131) reuses them, because its
  kernel/hardware slots hold the same values;
* step rows (features.py:143-172) are collected as (kind, value, axis)
  triples over the whole batch and written into ONE (ΣT, 6) array -- each
  ``StepSequence.steps`` is a row view into it, which is also the layout the
  device packer (csrc/host/tt_pack.c) copies fastest.

log2 uses ``math.log2`` (cached per value) so every element is bit-identical
to the reference's.  Errors are raised in record order with the reference's
messages: unresolvable task/target (features.py:175-186), the tile-slot cap
(features.py:113-117), the step-count bound (StepSequence, features.py:83-87),
labels of error records (features.py:201-204).

``make_encoders(features)`` binds the functions to a loaded reference
``features`` module (its StepSequence class and layout constants);
``install()`` patches them into ``tensortune.features/models/transfer``.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import DataValidationError

_LOG2: dict = {}


def _log2(v) -> float:
    r = _LOG2.get(v)
    if r is None:
        r = _LOG2[v] = math.log2(v)
    return r


class _Batch:
    """Shared per-call state: per-task context rows and label minima."""

    def __init__(self, features, ds):
        self.f = features
        # raise the bound reference module's own class (callers catch it by name)
        self.err = getattr(features, "DataValidationError", DataValidationError)
        self.ds = ds
        self.ctx_rows: list = []
        self.ctx_of: dict = {}
        self.tmin: dict = {}

    def resolve(self, rec):
        ds = self.ds
        task = ds.task_by_id.get(rec.task_id)
        if task is None:
            raise self.err(f"record {rec.record_id!r}: unresolvable task {rec.task_id!r}")
        hw = ds.hardware_by_id.get(task.target)
        if hw is None:
            raise self.err(f"record {rec.record_id!r}: unresolvable target {task.target!r}")
        return task, hw

    def context_index(self, task, hw) -> int:
        k = self.ctx_of.get(task.task_id)
        if k is None:
            k = self.ctx_of[task.task_id] = len(self.ctx_rows)
            self.ctx_rows.append(self.f.encode_context(task.kernel, hw))
        return k

    def label(self, rec) -> float:
        if rec.error_flag or rec.mean_cost is None:
            raise self.err(f"record {rec.record_id!r}: labels are undefined for error records")
        task, _ = self.resolve(rec)
        m = self.tmin.get(task.task_id, _MISSING)
        if m is _MISSING:
            costs = [r.mean_cost for r in self.ds.valid_records_of_task(task.task_id)
                     if r.mean_cost is not None]
            m = self.tmin[task.task_id] = min(costs) if costs else None
        c = rec.mean_cost
        best = c if m is None or c < m else m
        return best / c

    def contexts(self, idx) -> np.ndarray:
        table = np.asarray(self.ctx_rows, dtype=np.float64).reshape(len(self.ctx_rows), -1)
        return table[np.asarray(idx, dtype=np.int64)]


_MISSING = object()


def make_encoders(features):
    """(encode_sequence_batch, encode_flat_batch) over the reference's
    ``features`` module (layout constants and StepSequence class)."""
    SS = features.StepSequence
    kinds_n = len(features.STEP_KINDS)
    width = features.STEP_WIDTH
    max_steps = features.MAX_SEQUENCE_STEPS
    n_ops, n_dims = features.N_OPS, features.DIM_SLICE.stop - features.DIM_SLICE.start
    flat_len, tile0, max_tiles = features.FLAT_LENGTH, features.TILE_SLICE.start, features.MAX_TILE_SLOTS
    unroll_slot, vec_slot = features.UNROLL_SLOT, features.VECTORIZE_SLOT
    tx_slot, ty_slot = features.THREADS_X_SLOT, features.THREADS_Y_SLOT
    hwv, hwm = features.HW_VALUE_SLICE, features.HW_MASK_SLICE
    n_hw = hwv.stop - hwv.start
    TILE, UNROLL, VEC, BIND = (features.STEP_KINDS.index(k) for k in ("tile", "unroll", "vectorize", "bind"))

    def encode_sequence_batch(ds, record_ids):
        """features.py:229-238, batched."""
        b = _Batch(features, ds)
        n = len(record_ids)
        kinds: list = []
        vals: list = []
        axes: list = []
        lens = np.empty(n, dtype=np.int64)
        cidx = np.empty(n, dtype=np.int64)
        ys = np.empty(n, dtype=np.float64)
        for i, rid in enumerate(record_ids):
            rec = ds.record_by_id[rid]
            task, hw = b.resolve(rec)
            s = rec.schedule
            t0 = len(kinds)
            for axis, factors in enumerate(s.tile_factors):
                for fac in factors:
                    kinds.append(TILE)
                    vals.append(_log2(fac))
                    axes.append(float(axis))
            kinds.append(UNROLL)
            vals.append(_log2(s.unroll_factor))
            axes.append(-1.0)
            kinds.append(VEC)
            vals.append(_log2(s.vectorize_width))
            axes.append(-1.0)
            if s.thread_binding is not None:
                tx, ty = s.thread_binding
                kinds.extend((BIND, BIND))
                vals.extend((_log2(tx), _log2(ty)))
                axes.extend((0.0, 1.0))
            T = len(kinds) - t0
            cidx[i] = b.context_index(task, hw)
            if not 1 <= T <= max_steps:
                raise b.err(f"sequences must have 1..{max_steps} steps, got {T}")
            lens[i] = T
            ys[i] = b.label(rec)
        if n == 0:
            return [], ys
        R = len(kinds)
        steps = np.zeros((R, width), dtype=np.float64)
        steps[np.arange(R), np.asarray(kinds, dtype=np.int64)] = 1.0
        steps[:, kinds_n] = vals
        steps[:, kinds_n + 1] = axes
        ctx = b.contexts(cidx)
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        seqs = []
        new = SS.__new__
        for i in range(n):
            q = new(SS)
            q.steps = steps[off[i]:off[i + 1]]
            q.context = ctx[i]
            seqs.append(q)
        return seqs, ys

    def encode_flat_batch(ds, record_ids):
        """features.py:216-226, batched."""
        b = _Batch(features, ds)
        n = len(record_ids)
        rows = np.zeros((n, flat_len), dtype=np.float64)
        cidx = np.empty(n, dtype=np.int64)
        ys = np.empty(n, dtype=np.float64)
        for i, rid in enumerate(record_ids):
            rec = ds.record_by_id[rid]
            task, hw = b.resolve(rec)
            cidx[i] = b.context_index(task, hw)
            s = rec.schedule
            factors = [f for axis in s.tile_factors for f in axis]
            if len(factors) > max_tiles:
                raise b.err(
                    f"schedule has {len(factors)} tile factors, cap is {max_tiles}")
            r = rows[i]
            for j, fac in enumerate(factors):
                r[tile0 + j] = _log2(fac)
            r[unroll_slot] = _log2(s.unroll_factor)
            r[vec_slot] = _log2(s.vectorize_width)
            if s.thread_binding is not None:
                tx, ty = s.thread_binding
                r[tx_slot] = _log2(tx)
                r[ty_slot] = _log2(ty)
            ys[i] = b.label(rec)
        if n:
            ctx = b.contexts(cidx)
            k = n_ops + n_dims + 1          # op one-hot | dims | log flops
            rows[:, :k] = ctx[:, :k]
            rows[:, hwv] = ctx[:, k:k + n_hw]
            rows[:, hwm] = ctx[:, k + n_hw:k + 2 * n_hw]
        return rows, ys

    return encode_sequence_batch, encode_flat_batch
