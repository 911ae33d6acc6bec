"""GradientBoostedTrees on the GPU <- estimators/gbdt.py:51-265.

Same constructor, validation messages, ``fit(X, y, eval_set)`` /
``predict`` / ``get_weights`` / ``set_weights``, attributes
(``n_features_in_``, ``base_prediction_``, ``trees_``, ``train_curve_``)
and results -- bit for bit: every tree (node arrays in the reference's
stack order), every curve value and every prediction equal the reference's
(tests/test_gpu_gbdt.py against goldens made by the reference itself).

Per boosting round: one ``tt_gbdt_grow`` (csrc/tt_gbdt.cu: level-wise exact
split search over the sorted-index matrix, numpy's summation orders
reproduced), one ``tt_gbdt_update`` (pred += lr * incr; g = y - pred), the
validation rows advanced by the new tree with ``tt_gbdt_predict``, and the
curve's rmse from the downloaded predictions with the reference's own numpy
expression.  The stable per-column argsort is computed once on the host
(numpy's, as gbdt.py:109).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from sklearn.base import BaseEstimator, RegressorMixin

from . import _device, _lib
from .errors import DataValidationError, NumericFailure
from .estimators import _check_matrix


@dataclass
class _Tree:
    """One tree in the reference's layout (gbdt.py:19-38): node arrays in the
    order of the reference's growth stack, root 0, -1 at leaves."""

    feature: np.ndarray    # int32
    threshold: np.ndarray  # float64
    left: np.ndarray       # int32
    right: np.ndarray      # int32
    value: np.ndarray      # float64

    def predict(self, X: np.ndarray) -> np.ndarray:
        X = np.asarray(X, dtype=np.float64)
        return _predict_trees([self], 0.0, 1.0, X)


def _stack_order(feat, thr, left, right, val) -> _Tree:
    """Level-order arrays -> the reference's node numbering: ids are handed
    out when a node is popped and split (left, then right), the right child
    is popped first (gbdt.py:146-212)."""
    order = [0]
    new_of = np.full(feat.shape[0], -1, dtype=np.int64)
    new_of[0] = 0
    stack = [0]
    while stack:
        b = stack.pop()
        if feat[b] >= 0:
            lc, rc = int(left[b]), int(right[b])
            new_of[lc] = len(order)
            order.append(lc)
            new_of[rc] = len(order)
            order.append(rc)
            stack.append(lc)
            stack.append(rc)
    o = np.asarray(order, dtype=np.int64)
    L, R = left[o], right[o]
    return _Tree(feature=feat[o].astype(np.int32), threshold=thr[o].astype(np.float64),
                 left=np.where(L >= 0, new_of[np.maximum(L, 0)], -1).astype(np.int32),
                 right=np.where(R >= 0, new_of[np.maximum(R, 0)], -1).astype(np.int32),
                 value=val[o].astype(np.float64))


def _flat(trees):
    counts = np.asarray([t.feature.shape[0] for t in trees], dtype=np.int64)
    toff = np.zeros(len(trees) + 1, dtype=np.int64)
    np.cumsum(counts, out=toff[1:])
    cat = (lambda k, dt: np.concatenate([getattr(t, k) for t in trees]).astype(dt)  # noqa: E731
           if trees else np.zeros(0, dt))
    return (toff, cat("feature", np.int32), cat("threshold", np.float64), cat("left", np.int32),
            cat("right", np.int32), cat("value", np.float64))


def _predict_trees(trees, base: float, lr: float, X: np.ndarray, dev_cache=None) -> np.ndarray:
    t = _device.require_cuda()
    n, F = X.shape
    if n == 0:
        return np.zeros(0)
    if dev_cache is None:
        toff, feat, thr, left, right, val = _flat(trees)
        dev_cache = tuple(_device.to_dev(a) for a in (toff, feat, thr, left, right, val))
    dtoff, dfeat, dthr, dleft, dright, dval = dev_cache
    Xd = _device.to_dev(np.ascontiguousarray(X, dtype=np.float64))
    out = _device.empty(n, t.float64)
    if dfeat.numel() == 0:  # no trees: every row is the base prediction
        out.fill_(base)
        return out.cpu().numpy()
    _lib.call("tt_gbdt_predict", dfeat.data_ptr(), dthr.data_ptr(), dleft.data_ptr(), dright.data_ptr(),
              dval.data_ptr(), dtoff.data_ptr(), len(trees), float(base), float(lr), Xd.data_ptr(), n, F, 0,
              out.data_ptr(), 0, _device.stream_ptr())
    return out.cpu().numpy()


class GradientBoostedTrees(BaseEstimator, RegressorMixin):
    """Squared-error boosting with exact split search (gbdt.py:51-265)."""

    def __init__(
        self,
        num_trees: int = 200,
        max_depth: int = 6,
        learning_rate: float = 0.1,
        min_samples_leaf: int = 4,
    ) -> None:
        self.num_trees = num_trees
        self.max_depth = max_depth
        self.learning_rate = learning_rate
        self.min_samples_leaf = min_samples_leaf

    def _validate_params(self) -> None:
        if self.num_trees < 1:
            raise DataValidationError("num_trees must be >= 1")
        if self.max_depth < 1:
            raise DataValidationError("max_depth must be >= 1")
        if not 0.0 < self.learning_rate <= 1.0:
            raise DataValidationError("learning_rate must be in (0, 1]")
        if self.min_samples_leaf < 1:
            raise DataValidationError("min_samples_leaf must be >= 1")

    def fit(self, X, y, eval_set=None):
        self._validate_params()
        X = _check_matrix(X)
        y = np.asarray(y, dtype=np.float64)
        if y.ndim != 1 or y.shape[0] != X.shape[0]:
            raise DataValidationError("y must be 1-d and match X rows")
        if X.shape[0] < 1:
            raise DataValidationError("fit needs at least one sample")
        if not np.isfinite(y).all():
            raise DataValidationError("y contains non-finite values")
        X_val = y_val = None
        if eval_set is not None:
            X_val = _check_matrix(eval_set[0], "X_val")
            y_val = np.asarray(eval_set[1], dtype=np.float64)

        t = _device.require_cuda()
        n, F = X.shape
        self.n_features_in_ = F
        self.base_prediction_ = float(y.mean())
        self.trees_ = []
        self.train_curve_ = []
        self.__dict__.pop("_dev_tree_cache", None)
        lr = float(self.learning_rate)

        # per-feature stable argsort (gbdt.py:109) on the device: ties keep row
        # order as numpy's stable sort does; + 0.0 maps -0.0 to 0.0, which
        # numpy also treats as equal (a bit-pattern radix sort would not)
        d_X = _device.to_dev(np.ascontiguousarray(X))
        d_order = t.sort(d_X + 0.0, dim=0, stable=True).indices.to(t.int32).T.contiguous()
        d_Xc = d_X.T.contiguous()
        del d_X
        d_y = _device.to_dev(y)
        d_pred = _device.to_dev(np.full(n, self.base_prediction_))
        d_g = _device.empty(n, t.float64)
        st = _device.stream_ptr()
        _lib.call("tt_gbdt_update", d_pred.data_ptr(), None, d_y.data_ptr(), d_g.data_ptr(), 0.0, n, st)
        cap = 2 * n + 1
        d_feat = _device.empty(cap, t.int32)
        d_thr = _device.empty(cap, t.float64)
        d_left = _device.empty(cap, t.int32)
        d_right = _device.empty(cap, t.int32)
        d_val = _device.empty(cap, t.float64)
        d_cnt = _device.empty(1, t.int32)
        d_incr = _device.empty(n, t.float64)
        md = int(self.max_depth)
        nbytes = _lib.load().tt_gbdt_workspace_bytes(n, F, md)
        ws = _device.workspace(nbytes, "gbdt")
        d_toff0 = _device.to_dev(np.zeros(1, dtype=np.int64))
        d_Xv = d_vpred = None
        if X_val is not None and X_val.shape[0] > 0:
            d_Xv = _device.to_dev(np.ascontiguousarray(X_val))
            d_vpred = _device.to_dev(np.full(X_val.shape[0], self.base_prediction_))
        vp_host = np.full(0 if y_val is None else y_val.shape[0], self.base_prediction_)
        for _ in range(self.num_trees):
            _lib.call("tt_gbdt_grow", d_Xc.data_ptr(), d_g.data_ptr(), d_order.data_ptr(), n, F, md,
                      int(self.min_samples_leaf), d_feat.data_ptr(), d_thr.data_ptr(), d_left.data_ptr(),
                      d_right.data_ptr(), d_val.data_ptr(), d_cnt.data_ptr(), d_incr.data_ptr(), ws.data_ptr(),
                      nbytes, st)
            _lib.call("tt_gbdt_update", d_pred.data_ptr(), d_incr.data_ptr(), d_y.data_ptr(), d_g.data_ptr(),
                      lr, n, st)
            if d_Xv is not None:  # val_pred += lr * tree.predict(X_val), level-order arrays on device
                _lib.call("tt_gbdt_predict", d_feat.data_ptr(), d_thr.data_ptr(), d_left.data_ptr(),
                          d_right.data_ptr(), d_val.data_ptr(), d_toff0.data_ptr(), 1, 0.0, lr,
                          d_Xv.data_ptr(), X_val.shape[0], F, 0, d_vpred.data_ptr(), 1, st)
            k = int(d_cnt.item())
            tree = _stack_order(d_feat[:k].cpu().numpy(), d_thr[:k].cpu().numpy(), d_left[:k].cpu().numpy(),
                                d_right[:k].cpu().numpy(), d_val[:k].cpu().numpy())
            self.trees_.append(tree)
            pred = d_pred.cpu().numpy()
            train_rmse = float(np.sqrt(np.mean((y - pred) ** 2)))
            if not np.isfinite(train_rmse):
                raise NumericFailure(f"training diverged at round {len(self.trees_)}")
            val_rmse = None
            if y_val is not None:
                if d_vpred is not None:
                    vp_host = d_vpred.cpu().numpy()
                val_rmse = float(np.sqrt(np.mean((y_val - vp_host) ** 2)))
            self.train_curve_.append((train_rmse, val_rmse))
        return self

    def _dev_trees(self):
        cache = self.__dict__.get("_dev_tree_cache")
        if cache is None or cache[0] is not self.trees_ or cache[1] != len(self.trees_):
            arrays = tuple(_device.to_dev(a) for a in _flat(self.trees_))
            cache = (self.trees_, len(self.trees_), arrays)
            self.__dict__["_dev_tree_cache"] = cache
        return cache[2]

    def predict(self, X) -> np.ndarray:
        if not hasattr(self, "trees_"):
            raise DataValidationError("predict called before fit")
        X = _check_matrix(X)
        if X.shape[1] != self.n_features_in_:
            raise DataValidationError(f"expected {self.n_features_in_} features, got {X.shape[1]}")
        return _predict_trees(self.trees_, self.base_prediction_, float(self.learning_rate), X,
                              self._dev_trees() if X.shape[0] else None)

    def get_weights(self) -> dict[str, np.ndarray]:
        node_counts = np.asarray([t.feature.shape[0] for t in self.trees_], dtype=np.int64)
        cat = (lambda k, dt: np.concatenate([getattr(t, k) for t in self.trees_])  # noqa: E731
               if self.trees_ else np.zeros(0, dt))
        return {
            "base": np.asarray([self.base_prediction_]),
            "n_features": np.asarray([self.n_features_in_], dtype=np.int64),
            "node_counts": node_counts,
            "feature": cat("feature", np.int32),
            "threshold": cat("threshold", np.float64),
            "left": cat("left", np.int32),
            "right": cat("right", np.int32),
            "value": cat("value", np.float64),
        }

    def set_weights(self, weights: dict[str, np.ndarray]) -> None:
        self.base_prediction_ = float(weights["base"][0])
        self.n_features_in_ = int(weights["n_features"][0])
        self.trees_ = []
        off = 0
        for count in weights["node_counts"]:
            sl = slice(off, off + int(count))
            self.trees_.append(_Tree(feature=weights["feature"][sl].astype(np.int32),
                                     threshold=weights["threshold"][sl].astype(np.float64),
                                     left=weights["left"][sl].astype(np.int32),
                                     right=weights["right"][sl].astype(np.int32),
                                     value=weights["value"][sl].astype(np.float64)))
            off += int(count)
        self.train_curve_ = []
        self.__dict__.pop("_dev_tree_cache", None)

    def __getstate__(self):
        state = dict(self.__dict__)
        state.pop("_dev_tree_cache", None)
        return state
