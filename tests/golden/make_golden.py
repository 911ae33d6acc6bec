"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports tensortune from /root/reference/pkg/src (read-only; bytecode
writing disabled) and writes small .npz fixtures next to this file.  The
fixtures are committed; nothing at test time reads /root/reference.

Every fixture records the reference call that produced it:
  pca.npz       metrics.pairwise_comparison_accuracy on the generators of
                tests/test_metrics.py:52-63 (seed 0, 300 cases) and
                tests/test_acceptance.py:70-85 (seed 2024, 1000 cases) plus
                larger tie-heavy cases
  topk.npz      metrics.top_k_score, k in {1, min(5, n)}
  ranking.npz   estimators.mlp.ranking_grad (ties, no-pair batches)
  adam.npz      estimators.optim.Adam, 3 steps with a frozen tensor
  mlp.npz       CostMLP init/predict/loss_and_gradients/fit
  tuner.npz     RecurrentAttentionTuner init/predict/loss_and_gradients/
                fit/continue_fit (small and default sizes)
  sampling.npz  sampling.filter_invalid / task_weights / prune_dataset on
                benchmarks.pruning_benchmark-style data
  gbdt.npz      estimators.gbdt.GradientBoostedTrees fit (get_weights,
                train_curve_) and predict on the convergence benchmark's flat
                features plus tie-heavy / adjacent-double / tiny cases
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from tensortune.benchmarks import convergence_benchmark, pruning_benchmark  # noqa: E402
from tensortune.estimators.gbdt import GradientBoostedTrees  # noqa: E402
from tensortune.features import encode_flat_batch  # noqa: E402
from tensortune.estimators.mlp import CostMLP, ranking_grad  # noqa: E402
from tensortune.estimators.optim import Adam  # noqa: E402
from tensortune.estimators.tuner import RecurrentAttentionTuner  # noqa: E402
from tensortune.features import CONTEXT_LENGTH, STEP_WIDTH, StepSequence  # noqa: E402
from tensortune.metrics import pairwise_comparison_accuracy, top_k_score  # noqa: E402
from tensortune.sampling import (  # noqa: E402
    SamplerConfig,
    filter_invalid,
    prune_dataset,
    task_priority_order,
    task_weights,
)
from tensortune.workload import flop_count  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(np.asarray(v).nbytes for v in arrays.values()), "bytes raw")


def flat_cases(cases):
    ys = np.concatenate([c[0] for c in cases])
    ss = np.concatenate([c[1] for c in cases])
    off = np.zeros(len(cases) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(c[0]) for c in cases])
    return ys, ss, off


def gen_pca():
    cases = []
    rng = np.random.default_rng(0)  # test_metrics.py:52-63
    for _ in range(300):
        n = int(rng.integers(2, 65))
        if rng.random() < 0.5:
            y = rng.integers(0, 5, size=n).astype(float)
            s = rng.integers(0, 5, size=n).astype(float)
        else:
            y = rng.normal(size=n)
            s = rng.normal(size=n)
        cases.append((y, s))
    rng = np.random.default_rng(2024)  # test_acceptance.py:70-85
    for _ in range(1000):
        n = int(rng.integers(2, 65))
        y = rng.normal(size=n)
        s = rng.normal(size=n)
        if rng.random() < 0.5:
            y = np.round(y, 1)
            s = np.round(s, 1)
        cases.append((y, s))
    rng = np.random.default_rng(77)
    for n in (2, 3, 257, 1000, 1500, 3001):
        y = np.round(rng.normal(size=n), 2)
        s = np.round(rng.normal(size=n), 1)
        s[::7] = -0.0
        s[1::7] = 0.0
        cases.append((y, s))
    cases.append((np.array([3.0, 1.0, 2.0]), np.array([3.0, 2.0, 1.0])))
    cases.append((np.array([1.0, 1.0]), np.array([5.0, 5.0])))
    cases.append((np.array([1.0, 2.0]), np.array([1.0, 1.0])))
    ys, ss, off = flat_cases(cases)
    expected = np.array([pairwise_comparison_accuracy(y, s) for y, s in cases])
    save("pca.npz", y=ys, s=ss, offsets=off, pca=expected)


def gen_topk():
    rng = np.random.default_rng(5)
    cases = []
    for _ in range(200):
        n = int(rng.integers(1, 40))
        y = rng.uniform(0.05, 1.0, size=n)
        s = np.round(rng.normal(size=n), 1)  # many ties -> stable order matters
        cases.append((y, s))
    ys, ss, off = flat_cases(cases)
    k1 = np.array([top_k_score(y, s, 1) for y, s in cases])
    k5 = np.array([top_k_score(y, s, min(5, len(y))) for y, s in cases])
    save("topk.npz", y=ys, s=ss, offsets=off, top1=k1, top5=k5)


def gen_ranking():
    rng = np.random.default_rng(21)
    cases = []
    for n in (1, 2, 5, 12, 16, 16, 33):
        y = rng.normal(size=n)
        if n == 16:
            y = np.round(y, 0)
        cases.append((y, rng.normal(size=n)))
    cases.append((np.full(6, 0.5), np.arange(6.0)))
    ys, ss, off = flat_cases(cases)
    losses, grads = [], []
    for y, s in cases:
        l, g = ranking_grad(y, s)
        losses.append(l)
        grads.append(g)
    save("ranking.npz", y=ys, s=ss, offsets=off, loss=np.array(losses),
         grad=np.concatenate(grads))


def gen_adam():
    rng = np.random.default_rng(8)
    params = {"a": rng.normal(size=(5, 3)), "b": rng.normal(size=7), "c": rng.normal(size=4)}
    init = {k: v.copy() for k, v in params.items()}
    opt = Adam(params, 3e-3)
    steps = []
    for t in range(3):
        g = {k: rng.normal(size=v.shape) * (10.0 ** (t - 1)) for k, v in params.items()}
        if t == 1:
            g.pop("c")  # frozen in this step, counter still advances
        steps.append(g)
        opt.step(g)
    out = {}
    for k in init:
        out["init_" + k] = init[k]
        out["final_" + k] = params[k]
        for t, g in enumerate(steps):
            if k in g:
                out[f"g{t}_{k}"] = g[k]
    save("adam.npz", **out)


def gen_mlp():
    rng = np.random.default_rng(31)
    X = rng.normal(size=(32, 47))
    y = rng.uniform(0.1, 1.0, size=32)
    m = CostMLP(epochs=0, seed=3).fit(X, y)
    out = {"X": X, "y": y}
    for k, v in m.params_.items():
        out["init_" + k] = v.copy()
    out["pred"] = m.predict(X)
    for loss in ("rmse", "ranking"):
        m.loss = loss
        l, g = m.loss_and_gradients(X[:16], y[:16])
        out[f"{loss}_loss"] = np.array(l)
        for k, v in g.items():
            out[f"{loss}_g_{k}"] = v
    # short training trajectory (both losses)
    Xs = rng.normal(size=(40, 5))
    ys = rng.normal(size=40)
    Xv = rng.normal(size=(9, 5))
    yv = rng.normal(size=9)
    out["fit_X"], out["fit_y"], out["fit_Xv"], out["fit_yv"] = Xs, ys, Xv, yv
    for loss in ("rmse", "ranking"):
        f = CostMLP(epochs=3, batch_size=8, learning_rate=3e-3, loss=loss, seed=1).fit(
            Xs, ys, eval_set=(Xv, yv))
        for k, v in f.params_.items():
            out[f"fit_{loss}_{k}"] = v.copy()
        out[f"fit_{loss}_curve"] = np.array(f.train_curve_, dtype=np.float64)
    save("mlp.npz", **out)


def seqs_of(rng, lengths, d0=STEP_WIDTH, C=CONTEXT_LENGTH):
    return [StepSequence(steps=rng.normal(size=(t, d0)), context=rng.normal(size=C))
            for t in lengths]


def pack_seqs(seqs):
    steps = np.concatenate([s.steps for s in seqs])
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([s.steps.shape[0] for s in seqs])
    ctx = np.stack([s.context for s in seqs])
    return steps, off, ctx


def gen_tuner():
    out = {}
    rng = np.random.default_rng(3)
    # -- small model (hidden 4, 2 layers): full params and gradients -----------
    seqs = seqs_of(rng, (2, 5, 3, 4, 1, 9, 7, 12))
    y = rng.uniform(0.1, 0.9, size=len(seqs))
    st, off, cx = pack_seqs(seqs)
    out.update(small_steps=st, small_off=off, small_ctx=cx, small_y=y)
    m = RecurrentAttentionTuner(epochs=0, hidden_size=4, recurrent_layers=2, seed=1).fit(seqs, y)
    for k, v in m.params_.items():
        out["small_init_" + k] = v.copy()
    out["small_pred"] = m.predict(seqs)
    for loss in ("rmse", "ranking"):
        m.loss = loss
        l, g = m.loss_and_gradients(seqs, y)
        out[f"small_{loss}_loss"] = np.array(l)
        for k, v in g.items():
            out[f"small_{loss}_g_{k}"] = v
    # -- default model (hidden 32, 3 layers, seed 0) ---------------------------
    lens = rng.integers(1, 13, size=40)
    seqs = seqs_of(rng, lens)
    y = rng.uniform(0.1, 0.9, size=len(seqs))
    st, off, cx = pack_seqs(seqs)
    out.update(dflt_steps=st, dflt_off=off, dflt_ctx=cx, dflt_y=y)
    m = RecurrentAttentionTuner(epochs=0, seed=0).fit(seqs, y)
    names = list(m.params_)
    out["dflt_init_sum"] = np.array([m.params_[k].sum() for k in names])
    out["dflt_init_abs"] = np.array([np.abs(m.params_[k]).sum() for k in names])
    out["dflt_pred"] = m.predict(seqs)
    out["dflt_pred_chunk7"] = m.predict(seqs, chunk=7)
    for loss in ("rmse", "ranking"):
        m.loss = loss
        l, g = m.loss_and_gradients(seqs[:16], y[:16])
        out[f"dflt_{loss}_loss"] = np.array(l)
        out[f"dflt_{loss}_gnorm"] = np.array([np.linalg.norm(g[k]) for k in names])
        for k in ("head_W2", "head_b2", "attn_bq", "attn_bo", "lstm2_bw_b", "lstm0_fw_Wx"):
            out[f"dflt_{loss}_g_{k}"] = g[k]
    # -- training trajectory: fit + grouped curve + heads-only continue_fit ----
    lens = rng.integers(1, 6, size=14)
    seqs = seqs_of(rng, lens)
    y = rng.uniform(0.1, 0.9, size=len(seqs))
    st, off, cx = pack_seqs(seqs)
    out.update(fit_steps=st, fit_off=off, fit_ctx=cx, fit_y=y)
    grp = np.array([0] * 5 + [1] * 5 + [2] * 4)
    out["fit_groups"] = grp
    for loss in ("rmse", "ranking"):
        f = RecurrentAttentionTuner(epochs=2, batch_size=4, hidden_size=4, recurrent_layers=1,
                                    learning_rate=3e-3, loss=loss, seed=9)
        f.fit(seqs, y, eval_set=(seqs, y), eval_groups=list(grp))
        for k, v in f.params_.items():
            out[f"fit_{loss}_{k}"] = v.copy()
        out[f"fit_{loss}_curve"] = np.array(f.train_curve_, dtype=np.float64)
        head = set(f.param_groups()["head"])
        f.continue_fit(seqs, y, epochs=2, learning_rate=1e-3, trainable=head)
        for k, v in f.params_.items():
            out[f"cont_{loss}_{k}"] = v.copy()
        out[f"cont_{loss}_curve"] = np.array(
            [(a, np.nan if b is None else b, np.nan if c is None else c)
             for a, b, c in f.train_curve_], dtype=np.float64)
    save("tuner.npz", **out)


def dataset_arrays(ds):
    flops, cost, valid, off = [], [], [], [0]
    for task in ds.tasks:
        for rid in ds.records_by_task[task.task_id]:
            r = ds.record_by_id[rid]
            flops.append(int(r.measured_flops))
            cost.append(np.nan if r.mean_cost is None else float(r.mean_cost))
            valid.append(not r.error_flag)
        off.append(len(flops))
    return (np.array(flops, dtype=np.int64), np.array(cost), np.array(valid),
            np.array(off, dtype=np.int64))


def gen_sampling():
    out = {}
    ds = pruning_benchmark(seed=0, n_tasks=60, records_per_task=40)
    flops, cost, valid, off = dataset_arrays(ds)
    # inject exact throughput ties into task 0 so the t >= threshold edge is pinned
    out.update(flops=flops, cost=cost, valid=valid, offsets=off)
    rid_order = [rid for t in ds.tasks for rid in ds.records_by_task[t.task_id]]
    cases = [(0.1, 8), (0.0, 1), (0.25, 30), (0.5, 20), (0.9, 3), (0.37, 25)]
    for ci, (q, mr) in enumerate(cases):
        f = filter_invalid(ds, SamplerConfig(low_perf_quantile=q, min_records_per_task=mr))
        kept = {r.record_id for r in f.records}
        out[f"keep_{ci}"] = np.array([rid in kept for rid in rid_order])
        kt = {t.task_id for t in f.tasks}
        out[f"tkeep_{ci}"] = np.array([t.task_id in kt for t in ds.tasks])
        thr = []
        for t in ds.tasks:
            v = ds.valid_records_of_task(t.task_id)
            tp = np.asarray([r.measured_flops / r.mean_cost for r in v])
            thr.append(float(np.quantile(tp, q)) if len(v) else np.nan)
        out[f"thr_{ci}"] = np.array(thr)
    out["cases"] = np.array(cases, dtype=np.float64)
    w = task_weights(ds)
    out["weights"] = np.array([w[t.task_id] for t in ds.tasks])
    out["task_flops"] = np.array([flop_count(t.kernel) for t in ds.tasks], dtype=np.int64)
    out["task_ops"] = np.array([t.kernel.op for t in ds.tasks])
    prio = task_priority_order(ds)
    out["priority"] = np.array([[t.task_id for t in ds.tasks].index(x) for x in prio])
    pr, rep = prune_dataset(ds, SamplerConfig(target_fraction=0.55, seed=0))
    out["prune_order"] = np.array([[t.task_id for t in ds.tasks].index(x)
                                   for x in rep.sampled_task_order])
    out["prune_mass"] = np.array(rep.retained_weight_mass)
    out["prune_records_after"] = np.array(rep.records_after)
    # a synthetic tie-heavy set: equal throughputs straddling the cut
    tf = np.array([1000] * 10 + [2000] * 7 + [10**18 + 1] * 5, dtype=np.int64)
    tc = np.array([1e-4, 1e-4, 2e-4, 2e-4, 2e-4, 3e-4, 1e-4, 5e-4, 5e-4, 1e-4,
                   1e-4, 2e-4, 2e-4, 2e-4, 1e-4, 1e-4, 3e-4,
                   0.5, 0.25, 0.5, 1.0, 0.125])
    tv = np.ones(22, dtype=bool)
    tv[3] = False
    to = np.array([0, 10, 17, 22], dtype=np.int64)
    out.update(tie_flops=tf, tie_cost=tc, tie_valid=tv, tie_off=to)
    for qi, q in enumerate((0.1, 0.3, 0.5, 0.75, 0.99)):
        thr = []
        for t in range(3):
            idx = [i for i in range(to[t], to[t + 1]) if tv[i]]
            tp = np.asarray([int(tf[i]) / float(tc[i]) for i in idx])
            thr.append(float(np.quantile(tp, q)))
        out[f"tie_thr_{qi}"] = np.array(thr)
    out["tie_q"] = np.array((0.1, 0.3, 0.5, 0.75, 0.99))
    save("sampling.npz", **out)


def gen_gbdt():
    out = {}
    cases = []
    ds, a = convergence_benchmark(seed=0, n_tasks=6, records_per_task=40)
    Xtr, ytr = encode_flat_batch(ds, sorted(a.train_ids))
    Xte, yte = encode_flat_batch(ds, sorted(a.test_ids))
    cases.append(("conv", Xtr, ytr, Xte, yte, dict(num_trees=12, max_depth=4, learning_rate=0.1,
                                                      min_samples_leaf=4)))
    rng = np.random.default_rng(7)
    X = np.round(rng.normal(size=(300, 5)), 1)   # heavy ties: x[i] < x[i+1] gating
    y = rng.normal(size=300)
    cases.append(("ties", X, y, X[:50] + 0.05, y[:50], dict(num_trees=8, max_depth=6, learning_rate=0.3,
                                                             min_samples_leaf=2)))
    b = np.nextafter(1.0, 2.0)                   # (a + b) / 2 rounds to b: x <= cut takes both
    X = np.array([[1.0, 0.0], [b, 1.0], [1.0, 2.0], [b, 3.0], [2.0, 4.0], [1.0, 5.0]])
    y = np.array([0.0, 1.0, 0.2, 1.1, 3.0, 0.1])
    cases.append(("adjacent", X, y, X, y, dict(num_trees=3, max_depth=3, learning_rate=1.0,
                                                min_samples_leaf=1)))
    cases.append(("single", np.array([[0.5, 1.0]]), np.array([2.0]), np.array([[0.0, 0.0]]),
                  np.array([1.0]), dict(num_trees=2, max_depth=2, learning_rate=0.5, min_samples_leaf=1)))
    X = rng.normal(size=(2000, 12))
    y = np.sin(X[:, 0]) + 0.1 * rng.normal(size=2000)
    cases.append(("deep", X, y, X[:100], y[:100], dict(num_trees=4, max_depth=12, learning_rate=0.2,
                                                        min_samples_leaf=3)))
    for name, Xa, ya, Xb, yb, kw in cases:
        m = GradientBoostedTrees(**kw).fit(Xa, ya, eval_set=(Xb, yb))
        for k, v in m.get_weights().items():
            out[f"{name}_w_{k}"] = v
        out[f"{name}_curve"] = np.array([[t, np.nan if v is None else v] for t, v in m.train_curve_])
        out[f"{name}_pred"] = m.predict(Xb)
        out[f"{name}_X"], out[f"{name}_y"], out[f"{name}_Xv"], out[f"{name}_yv"] = Xa, ya, Xb, yb
        out[f"{name}_params"] = np.array([kw["num_trees"], kw["max_depth"], kw["learning_rate"],
                                          kw["min_samples_leaf"]], dtype=np.float64)
    out["names"] = np.array([c[0] for c in cases])
    save("gbdt.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()["gen_" + name]()
        sys.exit(0)
    gen_gbdt()
    gen_pca()
    gen_topk()
    gen_ranking()
    gen_adam()
    gen_mlp()
    gen_tuner()
    gen_sampling()
