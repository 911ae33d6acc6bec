"""GBDT restatement (TEST INFRASTRUCTURE ONLY) <- estimators/gbdt.py:51-265.

Squared-error boosting on residuals with exact greedy splits, restated the
way the GPU kernels (csrc/tt_gbdt.cu) build a tree -- level by level over a
per-feature sorted index matrix that is stably partitioned in place -- and
then renumbered into the reference's depth-first node order, so checking
this restatement against the reference's golden trees (tests/golden/
gbdt.npz) also checks that construction order does not matter.

Reference semantics kept bit for bit:
* the per-node gradient total is ``g[rows].sum()`` (numpy pairwise sum) over
  the node's rows in feature-0 order (gbdt.py:167-169);
* per feature, the prefix sums are a SEQUENTIAL cumulative sum over the
  node's rows sorted by that feature, score = c^2/nl + (G - c)^2/nr, a
  position is eligible iff x[i] < x[i+1] and both sides hold >= min_leaf
  rows; the first maximum wins (np.argmax), then the first feature wins
  (strict >) (gbdt.py:170-190);
* the cut is (x[pos] + x[pos+1]) / 2 and rows go left iff x <= cut
  (gbdt.py:191-199);
* leaves hold G / m; nodes are numbered in the order of the reference's
  LIFO stack (children ids at the parent's split, left then right pushed,
  right popped first) (gbdt.py:146-212);
* pred += lr * increment, residual = y - pred, curve rmse = sqrt(mean(.))
  (gbdt.py:112-131).
"""

from __future__ import annotations

import numpy as np


def _grow_levelwise(X, g, root_order, max_depth, min_leaf):
    n, F = X.shape
    order = root_order.copy()  # (F, n), partitioned in place per level
    # BFS node table
    feat, thr, left, right, val = [], [], [], [], []
    incr = np.zeros(n)

    def new():
        feat.append(-1)
        thr.append(0.0)
        left.append(-1)
        right.append(-1)
        val.append(0.0)
        return len(feat) - 1

    level = [(new(), 0, n)]  # (node, start, length)
    depth = 0
    while level:
        nxt = []
        for node, s, m in level:
            rows0 = order[0, s:s + m]
            G = g[rows0].sum()
            best = None
            if depth < max_depth and m >= 2 * min_leaf:
                for j in range(F):
                    idx = order[j, s:s + m]
                    x = X[idx, j]
                    c = np.cumsum(g[idx])[:-1]
                    nl = np.arange(1, m, dtype=np.float64)
                    nr = m - nl
                    sc = c ** 2 / nl + (G - c) ** 2 / nr
                    ok = (x[:-1] < x[1:]) & (nl >= min_leaf) & (nr >= min_leaf)
                    if not ok.any():
                        continue
                    sc = np.where(ok, sc, -np.inf)
                    p = int(np.argmax(sc))
                    if best is None or sc[p] > best[0]:
                        best = (sc[p], j, (x[p] + x[p + 1]) / 2.0)
            if best is None:
                val[node] = G / m
                incr[rows0] = G / m
                continue
            _, j, cut = best
            goes_left = np.zeros(n, dtype=bool)
            seg = order[j, s:s + m]
            goes_left[seg[X[seg, j] <= cut]] = True
            nl_rows = int(goes_left[rows0].sum())
            for f in range(F):
                col = order[f, s:s + m]
                mk = goes_left[col]
                order[f, s:s + m] = np.concatenate([col[mk], col[~mk]])
            feat[node], thr[node] = j, cut
            lid, rid = new(), new()
            left[node], right[node] = lid, rid
            nxt.append((lid, s, nl_rows))
            nxt.append((rid, s + nl_rows, m - nl_rows))
        level = nxt
        depth += 1
    return (np.array(feat, dtype=np.int32), np.array(thr), np.array(left, dtype=np.int32),
            np.array(right, dtype=np.int32), np.array(val)), incr


def dfs_renumber(feat, thr, left, right, val):
    """Level-order node arrays -> the reference's stack order (root = 0)."""
    new_of = {0: 0}
    order = [0]
    stack = [0]
    while stack:
        b = stack.pop()
        if feat[b] >= 0:
            for c in (left[b], right[b]):
                new_of[int(c)] = len(order)
                order.append(int(c))
            stack.append(int(left[b]))
            stack.append(int(right[b]))
    o = np.array(order)
    remap = lambda a: np.where(a >= 0, np.array([new_of.get(int(x), -1) for x in a]), -1).astype(np.int32)  # noqa: E731
    return (feat[o].astype(np.int32), thr[o], remap(left[o]), remap(right[o]), val[o])


def tree_predict(tree, X):
    feat, thr, left, right, val = tree
    node = np.zeros(X.shape[0], dtype=np.int64)
    while True:
        f = feat[node]
        act = f >= 0
        if not act.any():
            return val[node]
        r = np.nonzero(act)[0]
        gl = X[r, f[r]] <= thr[node[r]]
        node[r] = np.where(gl, left[node[r]], right[node[r]])


def fit(X, y, *, num_trees=200, max_depth=6, learning_rate=0.1, min_samples_leaf=4, eval_set=None):
    """Returns (base, trees (DFS-numbered tuples), curve)."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    base = float(y.mean())
    root = np.argsort(X, axis=0, kind="stable").astype(np.int64).T.copy()
    pred = np.full(y.shape[0], base)
    vp = None
    if eval_set is not None:
        Xv = np.asarray(eval_set[0], dtype=np.float64)
        yv = np.asarray(eval_set[1], dtype=np.float64)
        vp = np.full(yv.shape[0], base)
    trees, curve = [], []
    for _ in range(num_trees):
        tree_bfs, incr = _grow_levelwise(X, y - pred, root, max_depth, min_samples_leaf)
        tree = dfs_renumber(*tree_bfs)
        trees.append(tree)
        pred += learning_rate * incr
        tr = float(np.sqrt(np.mean((y - pred) ** 2)))
        va = None
        if vp is not None:
            vp += learning_rate * tree_predict(tree, Xv)
            va = float(np.sqrt(np.mean((yv - vp) ** 2)))
        curve.append((tr, va))
    return base, trees, curve


def predict(base, trees, learning_rate, X):
    out = np.full(np.asarray(X).shape[0], base)
    for t in trees:
        out += learning_rate * tree_predict(t, np.asarray(X, dtype=np.float64))
    return out
