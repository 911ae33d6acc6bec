"""Host-CPU timing of the UNMODIFIED reference (``tensortune`` staged in
baseline/_ref by tools/stage_reference.py), for bench.py's reference arm and
its ``cpu_baseline`` object.  Nothing here runs on the GPU and nothing in the
product package imports it.

* ``host_cores()``                -- logical CPUs usable by this process
  (sched_getaffinity) and the lscpu model line;
* ``reference_training(...)``     -- ``RecurrentAttentionTuner.continue_fit``
  (tuner.py:397-466) for one epoch over a bounded slice of the bench
  workload: the reference's own loop (pack, forward, rank loss, backward,
  Adam, the per-epoch train-set predict); timed at 1 BLAS thread and at the
  default thread count, the faster one reported ("best of host": the
  training is ONE sequential Adam chain, so more processes would change the
  algorithm);
* ``best_of_host_scoring(...)``   -- SURVEY.md §8d's CPU baseline
  procedure: P = #cores single-BLAS-thread processes started together
  (a barrier), each running the reference's own
  ``RecurrentAttentionTuner.predict`` / ``CostMLP.predict`` (F = 164) /
  ``pairwise_comparison_accuracy`` (n = 4096) on its own shard for a fixed
  duration; aggregate = sum of the per-process rates.

If baseline/_ref is missing, ``available()`` is False and bench.py falls
back to the float64 numpy port in oracle/ (kind "port").
"""

from __future__ import annotations

import multiprocessing as mp
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(ROOT, "baseline", "_ref")


def available() -> bool:
    return os.path.isfile(os.path.join(REF, "tensortune", "__init__.py"))


def _import_ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import tensortune  # noqa: F401

    return tensortune


def host_cores() -> dict:
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        n = os.cpu_count() or 1
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return {"logical_cpus": n, "model": model}


def _limit_threads(n):
    try:
        from threadpoolctl import threadpool_limits

        return threadpool_limits(n)
    except Exception:  # noqa: BLE001
        return None


def _ref_seqs(tt, steps, off, ctx):
    from tensortune.features import StepSequence

    return [StepSequence(steps[off[i]:off[i + 1]], ctx[i]) for i in range(len(off) - 1)]


def reference_training(steps, off, ctx, y, n_sample=1024, batch=16, seconds=12.0) -> dict:
    """One-epoch ``continue_fit`` of the reference over the first `n_sample`
    programs of the workload (rank loss, minibatch 16, lr 1e-3); repeated
    while under `seconds`; the faster of 1 BLAS thread / default threads."""
    tt = _import_ref()
    from tensortune.estimators import RecurrentAttentionTuner as RefTuner

    n_sample = min(n_sample, len(y))
    seqs = _ref_seqs(tt, steps, off[:n_sample + 1], ctx[:n_sample])
    yy = np.asarray(y[:n_sample], dtype=np.float64)
    best = None
    for threads in (1, None):
        lim = _limit_threads(threads) if threads else None
        try:
            est = RefTuner(batch_size=batch, epochs=0, loss="ranking", seed=0).fit(seqs[:2], yy[:2])
            t_end = time.perf_counter() + seconds / 2
            done, t_used, reps = 0, 0.0, 0
            while True:
                t0 = time.perf_counter()
                est.continue_fit(seqs, yy, epochs=1, learning_rate=1e-3)
                t_used += time.perf_counter() - t0
                done += n_sample
                reps += 1
                if time.perf_counter() > t_end:
                    break
        finally:
            if lim is not None:
                lim.__exit__(None, None, None)
        rate = done / t_used
        if best is None or rate > best["value"]:
            best = {"value": rate, "threads": threads or "default", "reps": reps, "seconds": t_used}
    cores = 1 if best["threads"] == 1 else host_cores()["logical_cpus"]
    return {"value": best["value"], "unit": "samples/s", "cores": cores, "kind": "reference",
            "sample": (f"reference tensortune RecurrentAttentionTuner.continue_fit, epochs=1, "
                       f"{n_sample}-program slice of the workload (rank loss, batch {batch}, lr 1e-3), "
                       f"{best['reps']} epochs in {best['seconds']:.1f} s, BLAS threads: "
                       f"{best['threads']} (faster of 1 and default)")}


# ------------------------------------------------------- best of host --


def _worker_init(barrier):
    global _BARRIER
    _BARRIER = barrier


def _score_worker(args):
    kind, rank, seconds, seed = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    lim = _limit_threads(1)
    tt = _import_ref()
    rng = np.random.default_rng(seed + rank)
    if kind == "tuner":
        from tensortune.estimators import RecurrentAttentionTuner as RefTuner

        sys.path.insert(0, ROOT)
        import bench

        st, of, cx, y, _ = bench.synth(n_tasks=1, per_task=1024, seed=seed + rank)
        seqs = _ref_seqs(tt, st, of, cx)
        est = RefTuner(epochs=0, seed=0).fit(seqs[:2], y[:2])
        est.predict(seqs[:64])
        unit_per_call = len(seqs)

        def call():
            est.predict(seqs)
    elif kind == "mlp":
        from tensortune.estimators import CostMLP as RefMLP

        X = rng.normal(size=(4096, 164))
        est = RefMLP(epochs=0, seed=0).fit(X[:4], rng.normal(size=4))
        est.predict(X[:16])
        unit_per_call = X.shape[0]

        def call():
            est.predict(X)
    else:  # pca
        from tensortune.metrics import pairwise_comparison_accuracy

        yv = rng.uniform(size=4096)
        sv = rng.normal(size=4096)
        pairwise_comparison_accuracy(yv[:64], sv[:64])
        unit_per_call = 4096 * 4095 // 2

        def call():
            pairwise_comparison_accuracy(yv, sv)
    _BARRIER.wait()
    t0 = time.perf_counter()
    done = 0
    while True:
        call()
        done += unit_per_call
        dt = time.perf_counter() - t0
        if dt >= seconds:
            break
    if lim is not None:
        lim.__exit__(None, None, None)
    return done / dt


def best_of_host_scoring(seconds=4.0, processes=None) -> dict:
    """P single-threaded processes, each on its own shard."""
    P = processes or host_cores()["logical_cpus"]
    ctx = mp.get_context("spawn")
    out = {"processes": P, "blas_threads_per_process": 1}
    units = {"tuner": ("reference RecurrentAttentionTuner.predict (defaults, T ~ bench histogram)",
                       "programs/s"),
             "mlp": ("reference CostMLP.predict, F = 164, 4096 rows per call", "programs/s"),
             "pca": ("reference pairwise_comparison_accuracy, n = 4096", "pairs/s")}
    for kind, (what, unit) in units.items():
        barrier = ctx.Barrier(P)
        with ctx.Pool(P, initializer=_worker_init, initargs=(barrier,)) as pool:
            rates = pool.map(_score_worker, [(kind, r, seconds, 100) for r in range(P)])
        out[kind] = {"value": float(np.sum(rates)), "unit": unit, "per_process_median": float(np.median(rates)),
                     "what": what}
    return out


if __name__ == "__main__":
    import json

    print(json.dumps({"host": host_cores(), "scoring": best_of_host_scoring(2.0)}, indent=1))
