"""Search-time batched scoring.

The reference's searches score ONE candidate per simulated-annealing step
(search.py:319, :349) and <= ``population`` per evolution generation
(search.py:392-410); ``tune`` walks the tasks one after another or on a
thread pool (search.py:512-576).  Every scorer call is therefore a tiny
GPU batch dominated by launch and host overhead.

This module batches ACROSS TASKS without changing a single decision of the
search: every task still runs the reference's own, unmodified
``run_search`` (its own seed from ``_task_seed``, its own RNG stream), each
in a worker thread, and their scorer calls meet at a cross-task batcher.
When every live search is waiting on its scorer, the batcher concatenates
the pending candidates of all tasks into one ``estimator.predict`` call --
one packing pass and one kernel launch for hundreds to thousands of
programs -- and hands each task its slice.  The kernels score every program
independently of its batch neighbours (bit-identical under re-batching,
tests/test_gpu_tuner.py::test_predict_padding_and_chunk_invariance), so
``tune``'s result is bit-identical to the reference's for any batch mix,
which keeps the reference's promise that results do not depend on ``jobs``
(search.py:523-525, test_search.py:387-402).

``make_schedule_scorer`` (models.py:364-378) returns a scorer that behaves
exactly like the reference's when called directly, plus the hooks the
batcher uses (``features`` / ``estimator``).  ``tune`` runs the batched
path when the factory's scorers are those; any other scorer (the
reference's test stubs, custom callables) runs the reference's own ``tune``
unchanged.  ``install()`` patches both names into ``tensortune``.
"""

from __future__ import annotations

import sys
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import replace

import numpy as np


def _ref(name: str):
    return sys.modules[name]


class BatchableScorer:
    """models.make_schedule_scorer's closure (models.py:364-378), split into
    ``features`` (encoding + hw rewrite, host) and the estimator's
    ``predict`` so several tasks' features can share one predict call."""

    def __init__(self, model, task, ds):
        models = _ref("tensortune.models")
        models._check_layout(model)
        self.model = model
        self.task = task
        self.hw = ds.hardware_of(task)
        self.estimator = model.estimator

    @property
    def kind(self) -> str:
        return "seq" if self.model.kind == "tuner" else "flat"

    def features(self, schedules):
        models = _ref("tensortune.models")
        if self.model.kind == "tuner":
            seqs = [models.encode_schedule_steps(self.task.kernel, s, self.hw) for s in schedules]
            return models._apply_rewrite_sequences(self.model, seqs)
        X = np.stack([models.encode_schedule(self.task.kernel, s, self.hw) for s in schedules])
        return models._apply_rewrite_flat(self.model, X)

    def __call__(self, schedules):
        if not schedules:
            return np.zeros(0)
        return self.estimator.predict(self.features(schedules))


def make_schedule_scorer(model, task, ds):
    """Drop-in for models.make_schedule_scorer (same validation, same scores)."""
    return BatchableScorer(model, task, ds)


class CrossTaskBatcher:
    """Gathers the scorer calls of concurrently running searches.

    ``live`` counts the searches that may still call their scorer; each has
    at most one call pending (the search blocks on it).  When pending ==
    live, one predict scores all pending candidates.  Flushes happen under
    the lock, in the thread of the last arrival."""

    def __init__(self, estimator, kind: str):
        self.est = estimator
        self.kind = kind
        self.cv = threading.Condition()
        self.live = 0
        self.pending: list[dict] = []
        self.calls = 0
        self.programs = 0
        self.error: BaseException | None = None

    def join(self):
        with self.cv:
            self.live += 1

    def leave(self):
        with self.cv:
            self.live -= 1
            self._maybe_flush()

    def score(self, feats, n: int):
        slot = {"f": feats, "n": n, "out": None}
        with self.cv:
            self.pending.append(slot)
            self._maybe_flush()
            while slot["out"] is None and self.error is None:
                self.cv.wait()
            if slot["out"] is None:
                raise RuntimeError("batched scoring failed in another search") from self.error
            return slot["out"]

    def _maybe_flush(self):
        if not self.pending or len(self.pending) < self.live:
            return
        batch, self.pending = self.pending, []
        try:
            if self.kind == "seq":
                allf = [s for b in batch for s in b["f"]]
            else:
                allf = np.concatenate([b["f"] for b in batch], axis=0)
            scores = np.asarray(self.est.predict(allf), dtype=np.float64)
            o = 0
            for b in batch:
                b["out"] = scores[o:o + b["n"]]
                o += b["n"]
            self.calls += 1
            self.programs += o
        except BaseException as exc:  # noqa: BLE001 - surfaced in every waiting search
            self.error = exc
        self.cv.notify_all()


class _BatchedScorer:
    def __init__(self, inner: BatchableScorer, batcher: CrossTaskBatcher):
        self.inner, self.batcher = inner, batcher

    def __call__(self, schedules):
        if not schedules:
            return np.zeros(0)
        return self.batcher.score(self.inner.features(schedules), len(schedules))


def tune(ds, task_ids, scorer_factory, oracle_fn, cfg, jobs: int = 1, space_factory=None,
         max_live: int = 4096):
    """search.tune (search.py:512-576) with cross-task batched scoring.

    Same validation, task order, per-task seeds, searches, top-k oracle
    measurement and result; ``jobs`` does not change the result (as in the
    reference) and no longer limits concurrency: up to ``max_live`` searches
    run at once so their scorer calls batch.  Falls back to the reference's
    own tune when the factory's scorers are not batchable."""
    search = _ref("tensortune.search")
    cfg.validate()
    for tid in task_ids:
        if tid not in ds.task_by_id:
            raise search.DataValidationError(f"tune: unknown task {tid!r}")
    ordered = search.task_priority_order(ds, task_ids)
    if not ordered:
        return _reference_tune()(ds, task_ids, scorer_factory, oracle_fn, cfg, jobs, space_factory)
    scorers = {}
    first = scorer_factory(ordered[0])
    if not isinstance(first, BatchableScorer):
        return _reference_tune()(ds, task_ids, scorer_factory, oracle_fn, cfg, jobs, space_factory)
    scorers[ordered[0]] = first
    make_space = space_factory or search.default_space
    batcher = CrossTaskBatcher(first.estimator, first.kind)

    def search_one(tid):
        batched = True
        try:
            sc = scorers.pop(tid, None) or scorer_factory(tid)
            if (isinstance(sc, BatchableScorer) and sc.estimator is first.estimator
                    and sc.kind == first.kind):
                sc = _BatchedScorer(sc, batcher)
            else:  # a different model for this task: its own unbatched calls
                batched = False
                batcher.leave()
            task = ds.task_by_id[tid]
            space = make_space(task.kernel, ds.hardware_of(task))
            return search.run_search(space, sc, replace(cfg, seed=search._task_seed(cfg.seed, tid)))
        finally:
            if batched:
                batcher.leave()

    results = {}
    width = max(1, min(len(ordered), int(max_live)))

    def run(tid):
        results[tid] = search_one(tid)

    # a search joins the batcher when a worker starts it; searches beyond
    # `width` join as workers free up (a flush waits only for running ones)
    with ThreadPoolExecutor(max_workers=width) as pool:
        futs = []
        for tid in ordered:
            futs.append(pool.submit(_joined, batcher, run, tid))
        for f in futs:
            f.result()
    entries = [_measure(search, ds, tid, results[tid], oracle_fn) for tid in ordered]
    out = search.TuneResult(
        entries=entries,
        total_oracle_calls=sum(e.oracle_calls for e in entries),
        total_best_cost=float(sum(e.best_cost for e in entries)),
        method=cfg.method,
        top_k=cfg.top_k,
        seed=cfg.seed,
    )
    out.scoring_stats = {"predict_calls": batcher.calls, "programs": batcher.programs}
    return out


def _joined(batcher, fn, tid):
    batcher.join()
    return fn(tid)


def _measure(search, ds, tid, result, oracle_fn):
    """tune_one's measurement half (search.py:540-560): oracle cost of the
    model's top-k, first-best wins."""
    task = ds.task_by_id[tid]
    hw = ds.hardware_of(task)
    best_cost, best_schedule, best_score, calls = float("inf"), None, 0.0, 0
    for candidate, score in zip(result.candidates, result.scores):
        bad = search.validity_check(candidate, task.kernel, hw)
        if bad:
            raise search.TensorTuneError(f"search produced an invalid candidate for {tid}: {bad}")
        cost = oracle_fn(task.kernel, candidate, hw)
        calls += 1
        if cost < best_cost:
            best_cost, best_schedule, best_score = cost, candidate, score
    if best_schedule is None:
        raise search.DataValidationError(f"tune: no valid candidate for task {tid!r}")
    return search.TaskTuneEntry(tid, best_schedule, best_cost, best_score, calls)


_ORIG_TUNE = None


def bind_reference() -> None:
    """Capture the reference's own tune (the fallback) before install() patches it."""
    global _ORIG_TUNE
    search = _ref("tensortune.search")
    if _ORIG_TUNE is None and search.tune is not tune:
        _ORIG_TUNE = search.tune


def _reference_tune():
    bind_reference()
    if _ORIG_TUNE is None:
        raise RuntimeError("the reference's tune is not available (patched before bind_reference)")
    return _ORIG_TUNE
