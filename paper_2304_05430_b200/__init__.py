"""paper_2304_05430_b200 -- B200-native hot path of the tensortune cost model.

Drop-in replacements with the reference's names (paths relative to
/root/reference/pkg/src/tensortune):

    RecurrentAttentionTuner, CostMLP, ranking_grad   estimators/tuner.py, mlp.py
    GradientBoostedTrees                             estimators/gbdt.py
    pairwise_comparison_accuracy, top_k_score,        metrics.py
    ranking_loss, rmse
    filter_invalid, task_weights, prune_dataset       sampling.py

``install()`` patches a loaded ``tensortune`` so its models/transfer/search/
CLI layers run on these kernels.  Compute lives in
libtt_b200.so (C ABI: include/tt_b200.h); there is no CPU fallback.
"""

from __future__ import annotations

from . import config
from .errors import DataValidationError, NumericFailure, TensorTuneError
from .estimators import CostMLP, RecurrentAttentionTuner, ranking_grad
from .gbdt import GradientBoostedTrees
from .metrics import (
    grouped_pca,
    pairwise_comparison_accuracy,
    pca_counts,
    ranking_loss,
    rmse,
    segmented_pca,
    top_k_score,
)

__all__ = [
    "config",
    "TensorTuneError",
    "DataValidationError",
    "NumericFailure",
    "RecurrentAttentionTuner",
    "CostMLP",
    "GradientBoostedTrees",
    "ranking_grad",
    "pairwise_comparison_accuracy",
    "pca_counts",
    "segmented_pca",
    "grouped_pca",
    "top_k_score",
    "ranking_loss",
    "rmse",
]
