"""Install the B200 path into a loaded reference package (tensortune).

The reference resolves its estimators and metrics as module globals at call
time, so assigning our objects to those names routes the
whole host stack -- train_tuner/train_mlp/load_model (models.py:231, :264,
:473-491), fine_tune's ``type(base)(**get_params())`` clone (transfer.py:211),
the search scorer (models.py:364-378) and the CLI -- through the kernels:

  tensortune.models / tensortune.estimators / tensortune
      RecurrentAttentionTuner, CostMLP           -> estimators.*
      GradientBoostedTrees                       -> gbdt.* (f3)
  tensortune.metrics / .models / .transfer / tensortune
      pairwise_comparison_accuracy, top_k_score  -> metrics.*
  tensortune.models.per_task_metrics             -> one batched K1 + K10 launch
  tensortune.transfer._grouped_pca               -> metrics.grouped_pca
  tensortune.sampling.filter_invalid             -> sampling.filter_invalid (K2)
  tensortune.features / .models / .transfer
      encode_sequence_batch, encode_flat_batch   -> featurize (batched labels)
  tensortune.models / .cli / tensortune
      make_schedule_scorer                       -> search.BatchableScorer
  tensortune.search / .cli / tensortune
      tune                                       -> search.tune (cross-task
                                                    batched scoring, f2)
  tensortune.data / .cli / .models / tensortune
      loads/load/dumps/save_dataset              -> dataio (native record
                                                    codec, f4)

``uninstall()`` restores the originals.
"""

from __future__ import annotations

import sys

import numpy as np

from . import estimators as _est
from . import dataio as _dataio
from . import featurize as _feat
from . import gbdt as _gbdt
from . import metrics as _met
from . import sampling as _samp
from . import search as _search

_saved: list = []


def _patch(module, name, value):
    if module is None or not hasattr(module, name):
        return
    _saved.append((module, name, getattr(module, name)))
    setattr(module, name, value)


def make_per_task_metrics(models):
    """Batched models.py:384-419: same rows, same order, one launch each for
    PCA and top-1/top-min(5,n) over all test tasks."""

    def per_task_metrics(model, ds, assignment):
        test_ids = models._usable_ids(ds, assignment.test_ids)
        if not test_ids:
            raise _met.DataValidationError("no labeled records on the test side")
        test_pred = np.asarray(models.predict_records(model, ds, test_ids), dtype=np.float64)
        _, y_test = models.encode_flat_batch(ds, test_ids)
        by_task: dict = {}
        for i, rid in enumerate(test_ids):
            by_task.setdefault(ds.record_by_id[rid].task_id, []).append(i)
        order = [t for t in ds.tasks if t.task_id in by_task]
        ranked = [t for t in order if len(by_task[t.task_id]) >= 2]
        res = {}
        if ranked:
            idx = np.concatenate([np.asarray(by_task[t.task_id]) for t in ranked])
            off = np.zeros(len(ranked) + 1, dtype=np.int64)
            off[1:] = np.cumsum([len(by_task[t.task_id]) for t in ranked])
            yy, pp = y_test[idx], test_pred[idx]
            _met._as_pair(yy, pp, min_n=1)
            if not np.all(np.maximum.reduceat(yy, off[:-1]) > 0):
                raise _met.DataValidationError("top_k_score needs a positive best label")
            pca = _met.segmented_pca(yy, pp, off)
            p1, best = _met.segmented_topk(yy, pp, off, 1)
            p5, _ = _met.segmented_topk(yy, pp, off, 5)
            for i, t in enumerate(ranked):
                res[t.task_id] = (float(pca[i]), float(p1[i]) / float(best[i]),
                                  float(p5[i]) / float(best[i]))
        rows = []
        for t in order:
            row = {"task_id": t.task_id, "n_records": len(by_task[t.task_id])}
            if t.task_id in res:
                a, b, c = res[t.task_id]
                row.update({"pairwise_accuracy": a, "top1": b, "top5": c})
            else:
                row.update({"pairwise_accuracy": None, "top1": None, "top5": None})
            rows.append(row)
        return rows

    return per_task_metrics


def install() -> None:
    """Route a loaded ``tensortune`` through the B200 kernels."""
    import tensortune  # noqa: F401  (must be importable)

    mods = {k: sys.modules.get(k) for k in (
        "tensortune", "tensortune.models", "tensortune.estimators", "tensortune.metrics",
        "tensortune.transfer", "tensortune.sampling", "tensortune.estimators.tuner",
        "tensortune.estimators.mlp")}
    # the defining modules too, so `from tensortune.estimators.tuner import
    # RecurrentAttentionTuner` (test_acceptance.py:28-29) resolves to ours
    for key in ("tensortune", "tensortune.models", "tensortune.estimators",
                "tensortune.estimators.tuner", "tensortune.estimators.mlp"):
        _patch(mods[key], "RecurrentAttentionTuner", _est.RecurrentAttentionTuner)
        _patch(mods[key], "CostMLP", _est.CostMLP)
    _patch(mods["tensortune.estimators.mlp"], "ranking_grad", _est.ranking_grad)
    import tensortune.estimators.gbdt  # noqa: F401

    for key in ("tensortune.models", "tensortune.estimators", "tensortune.estimators.gbdt"):
        _patch(sys.modules.get(key), "GradientBoostedTrees", _gbdt.GradientBoostedTrees)
    for key in ("tensortune", "tensortune.metrics", "tensortune.models", "tensortune.transfer"):
        _patch(mods[key], "pairwise_comparison_accuracy", _met.pairwise_comparison_accuracy)
        _patch(mods[key], "top_k_score", _met.top_k_score)
        _patch(mods[key], "ranking_loss", _met.ranking_loss)
    if mods["tensortune.models"] is not None:
        _patch(mods["tensortune.models"], "per_task_metrics",
               make_per_task_metrics(mods["tensortune.models"]))
    _patch(mods["tensortune.transfer"], "_grouped_pca", _met.grouped_pca)
    _patch(mods["tensortune.sampling"], "filter_invalid", _samp.filter_invalid)
    # search-time batched scoring (f2): tune batches its scorer calls across
    # tasks when the scorers come from make_schedule_scorer
    import tensortune.cli  # noqa: F401  (imports tune / make_schedule_scorer by name)
    import tensortune.search  # noqa: F401

    _search.bind_reference()
    for key in ("tensortune.models", "tensortune.cli", "tensortune"):
        _patch(sys.modules.get(key), "make_schedule_scorer", _search.make_schedule_scorer)
    for key in ("tensortune.search", "tensortune.cli", "tensortune"):
        _patch(sys.modules.get(key), "tune", _search.tune)
    # dataset I/O (f4): the native record codec behind the reference's names
    import tensortune.data  # noqa: F401

    _dataio.bind_reference()
    for name in ("loads_dataset", "load_dataset", "dumps_dataset", "save_dataset"):
        for key in ("tensortune.data", "tensortune.cli", "tensortune.models", "tensortune"):
            _patch(sys.modules.get(key), name, getattr(_dataio, name))
    import tensortune.features as features

    enc_seq, enc_flat = _feat.make_encoders(features)
    for key in ("tensortune.features", "tensortune.models", "tensortune.transfer"):
        _patch(sys.modules.get(key), "encode_sequence_batch", enc_seq)
        _patch(sys.modules.get(key), "encode_flat_batch", enc_flat)


def uninstall() -> None:
    while _saved:
        module, name, value = _saved.pop()
        setattr(module, name, value)
