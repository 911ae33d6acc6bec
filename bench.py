"""Benchmark of the B200 hot path on BASELINE.json configs[1]:

  attention-inspired cost model (RecurrentAttentionTuner defaults: 3 biLSTM
  layers, hidden 32, 2 heads, 2 attention passes) trained with the pairwise
  rank loss on 64 tasks x 4096 programs (262,144 samples), minibatch 16
  (paper Table 4), Adam lr 1e-3, float32, synthetic data.

A "step" is one training epoch: 16,384 minibatches of 16, each one forward,
rank loss, backward, fixed-order gradient reduction and fused Adam update --
one cooperative kernel launch per epoch.  ``value`` = optimizer-consumed
samples/s over K timed epochs with the dataset resident in HBM (device
timed, CUDA events on the launching stream, L2 flushed between epochs).
``e2e`` = the same metric through the public API
``RecurrentAttentionTuner.continue_fit(seqs, y, epochs=1)`` from host step
sequences: packing, pinned host->device copies, the epoch, the per-epoch
train-set scoring for the curve and the device->host reads.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the reference's algorithm on the host CPU (the
float64 numpy oracle port in oracle/, kind "port"; the reference is pure
Python and has no separate compiled form) on a bounded sample of the same
workload.  Under torchrun only rank 0 runs it.

Data: per program T ~ the step-count histogram measured on gen_dataset
(SURVEY.md §6.2, T in 4..10, mean 7.1); step rows = one-hot kind (4),
log2 knob in [0, 5], axis in {-1, 0, 1, 2}; context ~ N(0, 1) (35); labels
per task min(c)/c with c ~ LogNormal(-9, 0.5).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TASKS, PER_TASK, BATCH = 64, 4096, 16
T_HIST = {4: 35, 5: 196, 6: 457, 7: 516, 8: 469, 9: 291, 10: 46}
CPU_SAMPLE_SECONDS = 12.0


# ----------------------------------------------------------------- data --


def synth(n_tasks=N_TASKS, per_task=PER_TASK, seed=0):
    """Host CSR programs + labels (float64)."""
    rng = np.random.default_rng(seed)
    n = n_tasks * per_task
    ts = np.array(list(T_HIST))
    ps = np.array(list(T_HIST.values()), dtype=np.float64)
    lens = rng.choice(ts, size=n, p=ps / ps.sum())
    rows = int(lens.sum())
    steps = np.zeros((rows, 6))
    kind = rng.integers(0, 4, size=rows)
    steps[np.arange(rows), kind] = 1.0
    steps[:, 4] = rng.integers(0, 6, size=rows)
    steps[:, 5] = rng.integers(-1, 3, size=rows)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    ctx = rng.normal(size=(n, 35))
    # log-cost = a fixed function of the schedule steps and context + noise,
    # scaled to LogNormal(-9, 0.5); labels are task-normalised min(c)/c
    w_step = np.array([0.3, -0.2, 0.5, -0.4, 0.15, 0.1])
    row_score = steps @ w_step
    prog_score = np.add.reduceat(row_score, off[:-1]) / lens + 0.3 * ctx[:, 0]
    z = prog_score + 0.5 * rng.normal(size=n)
    z = (z - z.mean()) / z.std()
    cost = np.exp(-9.0 + 0.5 * z).reshape(n_tasks, per_task)
    y = (cost.min(axis=1, keepdims=True) / cost).ravel()
    return steps, off, ctx, y, lens


class Seq:
    __slots__ = ("steps", "context")

    def __init__(self, steps, context):
        self.steps = steps
        self.context = context


def as_seqs(steps, off, ctx):
    return [Seq(steps[off[i]:off[i + 1]], ctx[i]) for i in range(len(off) - 1)]


def train_flops(lens):
    """Algorithmic FLOPs of one training pass: 3 x forward, forward =
    134,656*T + 45,568 per program (default dims)."""
    return float(np.sum(3.0 * (134656.0 * lens + 45568.0)))


# --------------------------------------------------------------- clocks --


class Clocks:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self, gpu=0):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except Exception:  # noqa: BLE001
            return None
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 9 and r[0].strip() == str(gpu)]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        mx = float(rows[0][2])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------ reference --


def cpu_baseline(steps, off, ctx, y, seconds=CPU_SAMPLE_SECONDS):
    """The reference algorithm (float64 numpy port, oracle/tuner.py) training
    the same model with the same rank loss and batch size on the first
    minibatches of a permutation, single BLAS thread, for ~`seconds`."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # noqa: BLE001
        threadpool_limits = None
    from oracle import tuner as otuner
    from oracle.adam import AdamOracle

    seqs = as_seqs(steps, off, ctx)
    p = otuner.init_params(0)
    opt = AdamOracle(p, 1e-3)
    perm = np.random.default_rng(1).permutation(len(seqs))
    n_full = max(1, len(seqs) // BATCH)  # wrap around the sample's minibatches
    ctxm = threadpool_limits(1) if threadpool_limits else None
    done = 0
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < seconds:
        j = k % n_full
        b = perm[j * BATCH:(j + 1) * BATCH]
        _, g = otuner.loss_and_gradients(p, [seqs[i] for i in b], y[b], "ranking")
        opt.step(g)
        done += len(b)
        k += 1
    dt = time.perf_counter() - t0
    if ctxm is not None:
        ctxm.__exit__(None, None, None)
    return {"value": done / dt, "unit": "samples/s", "cores": 1, "kind": "port",
            "sample": f"{k} minibatches x {BATCH} samples ({done}) of the same workload, "
                      f"float64 numpy oracle port of tuner.py, 1 BLAS thread, {dt:.1f} s"}


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU implementation of the path --
    the unmodified tensortune (baseline/_ref) RecurrentAttentionTuner.continue_fit
    epoch over a bounded slice of the same workload, rank 0 only (the other
    ranks exit without work).  Falls back to the float64 numpy port in
    oracle/ when baseline/_ref was not staged."""
    if rank != 0:
        return
    import refbench

    steps, off, ctx, y, lens = synth(seed=0)
    vals, cb = [], None
    for i in range(args.warmup + args.steps):
        if refbench.available():
            r = refbench.reference_training(steps, off, ctx, y, n_sample=512,
                                            seconds=4.0 if i < args.warmup else 8.0)
        else:
            r = cpu_baseline(steps, off, ctx, y, seconds=max(2.0, CPU_SAMPLE_SECONDS / 4))
        if i >= args.warmup:
            vals.append(r["value"])
            cb = r
    v = float(np.mean(vals))
    cb = dict(cb, value=v)
    cb["host"] = refbench.host_cores()
    line = {
        "impl": "reference", "metric": "rank-loss train samples/sec", "value": v, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * 512 / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "attention tuner (3x biLSTM h32, 2 heads x 2 passes) rank-loss "
                               "training, 64 tasks x 4096 programs, batch 16, Adam; bounded sample: "
                               "one continue_fit epoch over a 512-program slice per step",
                   "global_batch": BATCH, "seq_len": int(lens.max()), "parallelism": "cpu"},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- B200 --


def flush_l2(buf):
    buf.fill_(1)


def survey_configs(est, dims, flat, l2, stream, n_steps16, prog, yd, prng):
    """The other SURVEY §8d configurations at their stated sizes (device-timed
    with CUDA events unless noted): C3 bulk scoring of 4 M programs, C4 PCA
    over 2,308 tasks x 4096 (half the tasks' labels rounded to 3 decimals
    for ties) and its log-uniform-size variant, C5 pruning statistics over
    64 x 4096 records and a heads-only fine-tuning epoch."""
    import torch

    from paper_2304_05430_b200 import _device, _lib
    from paper_2304_05430_b200 import metrics as gm
    from paper_2304_05430_b200.estimators import _bias_corrections
    from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms
    from paper_2304_05430_b200.sampling import filter_stats

    out = {}

    def ev_time(fn, reps=2):
        fn()
        ts = []
        for _ in range(reps):
            flush_l2(l2)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            ts.append((e0, e1))
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(b) for a, b in ts])) / 1e3

    # C3: 4 M programs, T from the generator histogram
    st, of, cx, _, ln = synth(n_tasks=1024, per_task=4096, seed=11)
    big = DevicePrograms(HostPrograms(st, of, cx), "fp32")
    del st, cx
    nb = big.n
    for prec, key in (("tf32", "c3_scoring_4M_tc_tf32_programs_per_s"),
                      ("fp32", "c3_scoring_4M_fp32_programs_per_s")):
        est.precision = prec
        out[key] = nb / ev_time(lambda: est._predict_programs(big, dims, flat))
    est.precision = "fp32"
    del big
    # C4: PCA over 2,308 tasks x 4096 (19.36 G pairs) and n_t log-uniform in [64, 4096]
    rng = np.random.default_rng(4)
    for name, sizes in (("c4_pca", np.full(2308, 4096)),
                        ("c4_pca_loguniform", np.exp(rng.uniform(np.log(64), np.log(4096), 2308)).astype(np.int64))):
        toff = np.zeros(len(sizes) + 1, dtype=np.int64)
        np.cumsum(sizes, out=toff[1:])
        yv = rng.uniform(0.05, 1.0, size=int(toff[-1]))
        for t in range(0, len(sizes), 2):
            yv[toff[t]:toff[t + 1]] = np.round(yv[toff[t]:toff[t + 1]], 3)
        yt = torch.tensor(yv, device="cuda")
        st_ = torch.randn(int(toff[-1]), dtype=torch.float64, device="cuda")
        gm.pca_counts(yt, st_, toff)
        torch.cuda.synchronize()
        dts = []
        for _ in range(3):
            t0 = time.perf_counter()
            gm.pca_counts(yt, st_, toff)
            dts.append(time.perf_counter() - t0)
        dt = float(np.median(dts))
        pairs = float(np.sum(sizes * (sizes - 1) / 2))
        out[f"{name}_pairs_per_s"] = pairs / dt
        out[f"{name}_tasks_per_s"] = len(sizes) / dt
    # C5: pruning statistics (K2) over 64 x 4096 records (wall, host arrays in,
    # masks out) and one heads-only fine-tuning epoch at B = 16
    n5 = N_TASKS * PER_TASK
    fl = rng.integers(1 << 20, 1 << 40, size=n5)
    co = rng.lognormal(-9, 0.5, size=n5)
    va = rng.uniform(size=n5) > 0.02
    poff = np.arange(0, n5 + 1, PER_TASK, dtype=np.int64)
    filter_stats(fl, co, va, poff, 0.1, 8)
    t0 = time.perf_counter()
    filter_stats(fl, co, va, poff, 0.1, 8)
    out["c5_prune_stats_records_per_s"] = n5 / (time.perf_counter() - t0)
    host = est.__dict__["_host"]
    heads = set(est.param_groups()["attention"]) | set(est.param_groups()["head"])
    mask = _device.to_dev(np.concatenate([np.full(host[k].size, k in heads, dtype=np.uint8)
                                          for k in dims["names"]]))
    fl_, mm, vv = flat.clone(), torch.zeros_like(flat), torch.zeros_like(flat)
    perm = _device.to_dev(prng.permutation(prog.n).astype(np.int32))
    corr = _device.to_dev(_bias_corrections(0, n_steps16))
    # continue_fit's heads-only path: frozen last-layer outputs once, then
    # attention + head steps (the timed region includes computing the cache)
    def heads_epoch():
        frozen = est._frozen_outputs(dims, fl_, prog)
        est._launch_train(dims, fl_, mm, vv, prog, yd, perm, BATCH, _lib.TT_MODE_TRAIN, 1e-3, corr,
                          mask, frozen)

    tt = ev_time(heads_epoch, reps=1)
    out["c5_heads_only_finetune_samples_per_s"] = prog.n / tt
    tt = ev_time(lambda: est._launch_train(dims, fl_, mm, vv, prog, yd, perm, BATCH, _lib.TT_MODE_TRAIN,
                                           1e-3, corr, mask), reps=1)
    out["c5_masked_full_step_samples_per_s"] = prog.n / tt
    return out


def dp_exchange_cost(n_tasks=4):
    """Fused data-parallel exchange measured on this one GPU:
    two ranks run concurrently on disjoint halves of the SMs, exchanging
    their gradient slices inside the training kernel, against two
    independent single-rank runs on the same halves (tools/dp_sim_bench.py
    has the longer version).  The transport is this GPU's memory, not
    NVLink."""
    import torch

    from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib
    from paper_2304_05430_b200.dist import FusedDataParallelTuner
    from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    parts = []
    for r in range(2):
        st, of, cx, yy, _ = synth(n_tasks=n_tasks, per_task=PER_TASK, seed=10 + r)
        e = RecurrentAttentionTuner(batch_size=BATCH, loss="ranking", seed=0)
        e.precision = "fp32"
        e._init_params()
        parts.append((e, DevicePrograms(HostPrograms(st, of, cx), "fp32"), _device.to_dev(yy, torch.float32)))
    n = parts[0][1].n
    steps = (n + BATCH - 1) // BATCH
    out = {}
    _lib.call("tt_tuner_train_set_grid", sms // 2)
    try:
        for name, groups in (("independent", [[p] for p in parts]), ("fused_dp2", [parts])):
            ranks = [rk for g in groups
                     for rk in FusedDataParallelTuner.local_group([a for a, _, _ in g], [b for _, b, _ in g],
                                                                  [c for _, _, c in g], BATCH)]
            streams = [torch.cuda.Stream() for _ in ranks]
            rng = np.random.default_rng(0)
            best = None
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for rk, s in zip(ranks, streams):
                    with torch.cuda.stream(s):
                        rk.run(rng.permutation(n), 1e-3)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            out[name] = best / steps * 1e6
            for rk in ranks:
                rk.close()
    finally:
        _lib.call("tt_tuner_train_set_grid", 0)
    return {"dp2_sim_us_per_step": out["fused_dp2"], "dp2_sim_independent_us_per_step": out["independent"],
            "dp2_sim_exchange_us_per_step": out["fused_dp2"] - out["independent"]}


def mlp_training(n=65536, F=164):
    """CostMLP.fit's epoch kernel (mlp.py:111-144) at the reference's
    minibatch of 16, device time of one launch (one epoch)."""
    import torch

    from paper_2304_05430_b200 import CostMLP, _device, _lib
    from paper_2304_05430_b200.estimators import _bias_corrections

    rng = np.random.default_rng(3)
    X = rng.normal(size=(n, F))
    y = rng.uniform(0.1, 0.9, size=n)
    m = CostMLP(epochs=0, batch_size=BATCH, loss="ranking", seed=0)
    m.precision = "fp32"
    m.fit(X[:64], y[:64])
    flat = m._device_flat(list(m.NAMES)).clone()
    mm, vv = torch.zeros_like(flat), torch.zeros_like(flat)
    Xd = _device.to_dev(X.ravel(), torch.float32)
    yd = _device.to_dev(y, torch.float32)
    order = _device.to_dev(rng.permutation(n).astype(np.int32))
    steps = (n + BATCH - 1) // BATCH
    corr = _device.to_dev(_bias_corrections(0, steps))
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m._launch_train(flat, mm, vv, Xd, yd, F, order, BATCH, _lib.TT_MODE_TRAIN, 1e-3, corr)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.median(ts))
    return {"mlp_train_f164_samples_per_s": n / t, "mlp_train_us_per_step": t / steps * 1e6}


def mlp_scoring(l2, stream, peaks, n=4 * 1024 * 1024, F=164):
    """CostMLP bulk scoring at TenSet width (configs[0]/[2] shape): the
    tcgen05 kernels -- "fp32" (the default: split-precision tf32 at fp32
    accuracy) and "tf32" -- and the fp32 CUDA-core kernel ("fp32_cuda"), HBM
    roofline (algorithmic bytes 4F + 4 per row)."""
    import torch

    from paper_2304_05430_b200 import CostMLP, _lib

    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(n, F, device="cuda", generator=g)
    est = CostMLP(epochs=0, seed=0)
    est._init_params(F)
    out = {}
    for prec, fn in (("tf32", "tt_mlp_predict_tf32"), ("fp32", "tt_mlp_predict_f32tc"),
                     ("fp32_cuda", "tt_mlp_predict_f32")):
        est.precision = prec
        flat = est._device_flat(list(est.NAMES))
        y = torch.empty(n, device="cuda")
        for _ in range(3):
            _lib.call(fn, flat.data_ptr(), X.data_ptr(), n, F, y.data_ptr(), stream.cuda_stream)
        ts = []
        for _ in range(5):
            flush_l2(l2)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _lib.call(fn, flat.data_ptr(), X.data_ptr(), n, F, y.data_ptr(), stream.cuda_stream)
            e1.record(stream)
            ts.append((e0, e1))
        torch.cuda.synchronize()
        t = float(np.mean([a.elapsed_time(b) for a, b in ts])) / 1e3
        gbs = n * (4 * F + 4) / t / 1e9
        out[f"mlp_{prec}_rows_per_s"] = n / t
        out[f"mlp_{prec}_hbm_gbs"] = gbs
        out[f"mlp_{prec}_hbm_frac"] = gbs / float(peaks.get("hbm_gbs", 6552.0))
    return out


def allreduce_max(dist, x: float) -> float:
    """MAX of one float over the ranks (a CUDA tensor under NCCL, CPU under gloo)."""
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    v = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return float(v.item())


def sharded_extra(world, rank, dist, l2, stream, est, dims, flat):
    """Configs 3 and 4 across the ranks (SURVEY §8e, weak scaling): every rank
    scores its own 1 M-program shard (no collective on the data path), and the
    2,308-task PCA is split by LPT with one int64 all-reduce of the counts.
    Device time per rank (CUDA events), MAX over ranks."""
    import torch

    from paper_2304_05430_b200 import dist as tdist
    from paper_2304_05430_b200 import metrics as gm
    from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms

    def tmax(t):
        return allreduce_max(dist, t)

    out = {}
    st, of, cx, _, _ = synth(n_tasks=256, per_task=4096, seed=100 + rank)
    shard = DevicePrograms(HostPrograms(st, of, cx), "fp32")
    for prec in ("fp32", "tf32"):
        est.precision = prec
        est._predict_programs(shard, dims, flat)
        flush_l2(l2)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        est._predict_programs(shard, dims, flat)
        e1.record(stream)
        torch.cuda.synchronize()
        t = tmax(e0.elapsed_time(e1) / 1e3)
        out[f"c3_sharded_{prec}_programs_per_s"] = world * shard.n / t
    est.precision = "fp32"
    del shard
    rng = np.random.default_rng(4)
    sizes = np.full(2308, 4096)
    toff = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=toff[1:])
    yv = rng.uniform(0.05, 1.0, size=int(toff[-1]))
    sv = rng.normal(size=int(toff[-1]))
    tdist.sharded_pca_counts(yv, sv, toff)
    dist.barrier()
    t0 = time.perf_counter()
    c = tdist.sharded_pca_counts(yv, sv, toff)  # count + the one all-reduce, wall incl. host plan
    t = tmax(time.perf_counter() - t0)
    out["c4_sharded_pca_pairs_per_s"] = float(np.sum(sizes * (sizes - 1) / 2)) / t
    out["c4_sharded_pca_checksum"] = int(np.sum(c))
    out["c3_c4_ranks"] = world
    return out


def gbdt_fit_throughput(n=16384, F=164, trees=20, depth=6):
    """GradientBoostedTrees.fit (bit-exact trees, csrc/tt_gbdt.cu)
    on a synthetic TenSet-width matrix, wall clock through the estimator (the
    host drives the level loop), against the unmodified reference's fit on
    the same data for a bounded number of trees (per-tree cost is flat).
    Trees per second, and identical trees / predictions checked."""
    import refbench

    from paper_2304_05430_b200 import GradientBoostedTrees

    rng = np.random.default_rng(0)
    X = rng.normal(size=(n, F))
    y = np.tanh(X[:, 0] - 0.5 * X[:, 1] * X[:, 2]) + 0.05 * rng.normal(size=n)
    GradientBoostedTrees(num_trees=2, max_depth=depth).fit(X[:1024], y[:1024])  # warm
    t0 = time.perf_counter()
    g = GradientBoostedTrees(num_trees=trees, max_depth=depth).fit(X, y)
    t_gpu = time.perf_counter() - t0
    out = {"gbdt_fit_rows": n, "gbdt_fit_features": F, "gbdt_fit_depth": depth,
           "gbdt_fit_trees_per_s": trees / t_gpu}
    if refbench.available():
        refbench._import_ref()
        from tensortune.estimators.gbdt import GradientBoostedTrees as RefGBDT

        k = 2
        t0 = time.perf_counter()
        r = RefGBDT(num_trees=k, max_depth=depth).fit(X, y)
        t_ref = time.perf_counter() - t0
        g2 = GradientBoostedTrees(num_trees=k, max_depth=depth).fit(X, y)
        out.update({"gbdt_fit_reference_trees_per_s": k / t_ref,
                    "gbdt_fit_speedup_vs_reference": (trees / t_gpu) / (k / t_ref),
                    "gbdt_fit_identical_predictions": bool(np.array_equal(g2.predict(X[:4096]),
                                                                          r.predict(X[:4096])))})
    return out


def search_throughput(n_tasks=64, steps=128):
    """Search-time scoring (SURVEY §8 f2, config 3's real caller): the
    reference's tune (simulated annealing, one candidate per scorer call)
    with (a) the reference's own CPU tuner on a few tasks, (b) the GPU tuner
    through the reference's unbatched scorer, (c) the cross-task batched tune
    (paper_2304_05430_b200.search) -- whose result must be identical to (b).
    Wall clock (host search loop included): scored candidates per second."""
    import refbench

    if not refbench.available():
        return {}
    tt = refbench._import_ref()  # noqa: F841
    import tensortune.cli  # noqa: F401
    import tensortune.models as tm
    import tensortune.search as ts
    from tensortune.benchmarks import convergence_benchmark
    from tensortune.estimators import RecurrentAttentionTuner as RefTuner
    from tensortune.features import encode_sequence_batch
    from tensortune.oracle import OracleConfig, oracle_cost

    from paper_2304_05430_b200 import RecurrentAttentionTuner
    from paper_2304_05430_b200 import search as bs

    ds, a = convergence_benchmark(seed=0, n_tasks=n_tasks, records_per_task=24)
    seqs, y = encode_sequence_batch(ds, sorted(a.train_ids))
    est = RecurrentAttentionTuner(epochs=1, seed=0).fit(seqs, y)
    model = tm.CostModel(kind="tuner", estimator=est, config=tm.TrainConfig(epochs=1))
    ocfg = OracleConfig(noise_sigma=0.05, seed=0)

    def oracle_fn(k, sc, hw):
        return oracle_cost(k, sc, hw, ocfg)

    tids = [t.task_id for t in ds.tasks]
    cfg = ts.SearchConfig(method="anneal", steps=steps, top_k=8, seed=0)
    bs.bind_reference()
    out = {}
    t0 = time.perf_counter()
    r_unb = ts.tune(ds, tids, lambda t: tm.make_schedule_scorer(model, ds.task_by_id[t], ds), oracle_fn, cfg)
    t_unb = time.perf_counter() - t0
    t0 = time.perf_counter()
    r_bat = bs.tune(ds, tids, lambda t: bs.make_schedule_scorer(model, ds.task_by_id[t], ds), oracle_fn, cfg)
    t_bat = time.perf_counter() - t0
    n_scored = r_bat.scoring_stats["programs"]
    ref_model = tm.CostModel(kind="tuner", estimator=RefTuner(epochs=0, seed=0).fit(seqs[:2], y[:2]),
                             config=tm.TrainConfig(epochs=0))
    ref_model.estimator.set_weights(est.get_weights())
    few = tids[:4]
    n_cpu = [0]

    def cpu_factory(t):
        inner = tm.make_schedule_scorer(ref_model, ds.task_by_id[t], ds)

        def scorer(schedules):
            n_cpu[0] += len(schedules)
            return inner(schedules)
        return scorer

    t0 = time.perf_counter()
    ts.tune(ds, few, cpu_factory, oracle_fn, cfg)
    t_cpu = time.perf_counter() - t0
    out.update({
        "search_tasks": n_tasks, "search_sa_steps": steps, "search_candidates_scored": n_scored,
        "search_identical_to_reference_tune": r_bat.to_json() == r_unb.to_json(),
        "search_gpu_unbatched_candidates_per_s": n_scored / t_unb,
        "search_gpu_batched_candidates_per_s": n_scored / t_bat,
        "search_gpu_batched_predict_calls": r_bat.scoring_stats["predict_calls"],
        "search_reference_cpu_candidates_per_s_4_tasks": n_cpu[0] / t_cpu,
        "search_batched_speedup_vs_unbatched": t_unb / t_bat,
    })
    return out


def print_phases(est, dims, flat, m, v, prog, yd, rng, n, n_steps, t_adam, batch=BATCH):
    """Per-phase marks of one minibatch inside the train kernel (CTA 0 clock64
    at 1965 MHz; the first gradient-job CTA in %globaltimer ns)."""
    import ctypes

    import torch

    from paper_2304_05430_b200 import _device, _lib
    from paper_2304_05430_b200.estimators import _bias_corrections

    lib = _lib.load()
    names = {0: "start", 1: "adam_wait", 2: "fwd_l0", 3: "fwd_l1", 4: "fwd_l2", 8: "attn_kv",
             9: "attn_p0", 17: "attn_p1", 5: "head", 6: "yhat_xchg", 7: "loss", 18: "head_bwd",
             19: "attn_bwd_p1", 24: "attn_bwd_p0", 10: "dS", 11: "bptt_l2", 12: "dX_l2",
             13: "bptt_l1", 14: "dX_l1", 15: "bptt_l0", 16: "bwd_end"}
    for probe in (40, 41, 42):
        lib.tt_debug_profile_step(probe)
        buf0 = (ctypes.c_int64 * 32)()
        ctypes.memmove(buf0, (ctypes.c_int64 * 32)(), 32 * 8)
        perm = _device.to_dev(rng.permutation(n).astype(np.int32))
        corr = _device.to_dev(_bias_corrections(t_adam, n_steps))
        est._launch_train(dims, flat, m, v, prog, yd, perm, batch, _lib.TT_MODE_TRAIN, 1e-3, corr, None)
        t_adam += n_steps
        torch.cuda.synchronize()
        buf = (ctypes.c_int64 * 32)()
        lib.tt_debug_phase_times(buf, 32)
        mk = list(buf)
        prev = mk[0]
        row = []
        for i in sorted(names, key=lambda i: mk[i] if mk[i] else 0):
            if i == 0 or mk[i] == 0 or mk[i] < mk[0]:
                continue
            row.append(f"{names[i]}={(mk[i] - prev) / 1965.0:.2f}")
            prev = mk[i]
        last = max((i for i in names if mk[i] >= mk[0] and mk[i] != 0), key=lambda i: mk[i])
        jobs = ""
        if mk[20] and mk[30]:
            jobs = (f" | job CTA: start-after-cta0-bwd={(mk[20] - mk[30]) / 1e3:.2f}us "
                    f"stage={(mk[22] - mk[20]) / 1e3:.2f} compute={(mk[23] - mk[22]) / 1e3:.2f} "
                    f"adam+signal={(mk[21] - mk[23]) / 1e3:.2f}us")
        proj = " proj=" + ",".join(f"{(mk[25 + l] - mk[1 + l] if l == 0 else mk[25 + l] - mk[1 + l]) / 1965.0:.2f}"
                                  for l in range(3) if mk[25 + l])
        print(f"step {probe}: cta0 {(mk[last] - mk[0]) / 1965.0:.2f}us | " + " ".join(row) + proj + jobs,
              flush=True)
    lib.tt_debug_profile_step(-1)


def run_b200(args, world, rank):
    import torch

    from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib
    from paper_2304_05430_b200.estimators import _bias_corrections
    from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    if args.profile:  # small dataset for ncu replays (same kernels, fewer minibatches)
        steps, off, ctx, y, lens = synth(n_tasks=1, per_task=2048, seed=rank)
    else:
        steps, off, ctx, y, lens = synth(seed=rank)
    n = len(y)
    host = HostPrograms(steps, off, ctx)
    prog = DevicePrograms(host, "fp32")
    yd = _device.to_dev(y, torch.float32)
    est = RecurrentAttentionTuner(batch_size=BATCH, loss="ranking", seed=0)
    est.precision = "fp32"
    est._init_params()
    dims = est._dims()
    flat = est._dev_params(dims).clone()
    m = torch.zeros_like(flat)
    v = torch.zeros_like(flat)
    rng = np.random.default_rng(1)
    n_steps = (n + BATCH - 1) // BATCH
    l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    dp = None
    dp_kind = "none"
    if world > 1:
        # data parallel: every rank holds its own 64x4096 shard (weak scaling);
        # global step = the ranks' microbatches of 16 (SURVEY §8e option A),
        # exchanged inside the one training launch per epoch over NVLink peer
        # memory (paper_2304_05430_b200.dist.FusedDataParallelTuner)
        from paper_2304_05430_b200.dist import DataParallelTunerEpoch, FusedDataParallelTuner

        try:
            dp = FusedDataParallelTuner.create(est, prog, yd, BATCH)
            dp_kind = "fused peer-memory exchange in the training kernel"
        except Exception as exc:  # noqa: BLE001  (no P2P/IPC between the GPUs)
            print(f"fused DP unavailable ({exc}); NCCL all-reduce path", file=sys.stderr)
            dp = DataParallelTunerEpoch(est, prog, yd, BATCH)
            dp_kind = "NCCL all-reduce + Adam launch per step"

    def dp_epoch():
        if isinstance(dp, DataParallelTunerEpoch):
            dp.run(rng.permutation(n), 1e-3, local_shard=True)
            return None
        return dp.run(rng.permutation(n), 1e-3)

    def epoch(t0):
        if dp is not None:
            return dp_epoch()
        perm = _device.to_dev(rng.permutation(n).astype(np.int32))
        corr = _device.to_dev(_bias_corrections(t0, n_steps))
        return est._launch_train(dims, flat, m, v, prog, yd, perm, BATCH, _lib.TT_MODE_TRAIN, 1e-3,
                                 corr, None)

    t_adam = 0
    for _ in range(args.warmup):
        epoch(t_adam)
        t_adam += n_steps
    torch.cuda.synchronize()
    if args.phases and dp is None:
        print_phases(est, dims, flat, m, v, prog, yd, rng, n, n_steps, t_adam, args.phase_batch)
        t_adam += 3 * n_steps
    # pre-stage the timed epochs' inputs so the timed region holds only kernels
    perms = [_device.to_dev(rng.permutation(n).astype(np.int32)) for _ in range(args.steps)]
    corrs = [_device.to_dev(_bias_corrections(t_adam + k * n_steps, n_steps)) for k in range(args.steps)]
    times = []
    clocks = Clocks(os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")
                    if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else f"/tmp/clocks_{rank}.csv")
    with clocks:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush_l2(l2)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if dp is not None:
                status = dp_epoch()
            else:
                _, status, _ = est._launch_train(dims, flat, m, v, prog, yd, perms[k], BATCH,
                                                 _lib.TT_MODE_TRAIN, 1e-3, corrs[k], None)
            e1.record(stream)
            times.append((e0, e1))
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    ms = [a.elapsed_time(b) for a, b in times]
    assert status is None or int(status.cpu()[0]) < 0, "non-finite loss during the benchmark"
    if status is not None and status.numel() > 1:
        from paper_2304_05430_b200.dist import FusedDataParallelTuner

        FusedDataParallelTuner.check_status(status)
    t_mean = float(np.mean(ms)) / 1e3
    if dist is not None:
        t_mean = allreduce_max(dist, t_mean)
    value = world * n / t_mean
    flops = train_flops(lens)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        pass
    peak = float(peaks.get("bf16_tflops_sustained", 1400.0))
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "train_kernel_traffic.json")))
        traffic = prof.get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        pass
    achieved = flops / t_mean / 1e12
    # The B = 16 epoch is a chain of n_steps DEPENDENT Adam steps: its bound
    # is the per-step critical path, not a throughput pipe.  Reported: the
    # critical-path model (steps x measured per-step latency) and the FLOP
    # rate against the pipe the kernel actually issues on -- FP32 CUDA cores
    # (no tensor instructions in its SASS): 148 SMs x 128 lanes x 2 x clock.
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    clk_ghz = float(peaks.get("sm_max_mhz", 1965.0)) / 1e3
    fp32_peak = sm * 128 * 2 * clk_ghz / 1e3  # TFLOP/s
    roof = {"bound": "latency", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
            "frac": achieved / fp32_peak, "traffic": traffic,
            "kernel": "tuner_train_fast_kernel (latency path, one launch = one epoch)",
            "peak_source": f"FP32 CUDA-core issue peak {sm} SMs x 128 x 2 x {clk_ghz:.3f} GHz "
                           "(the kernel issues no tensor-core instructions)",
            "critical_path": {"dependent_adam_steps": n_steps,
                              "us_per_step": t_mean / n_steps * 1e6,
                              "model": "epoch = dependent steps x per-step latency (forward 3 layers + "
                                       "attention, loss exchange, backward, gradient jobs + Adam hand-off)"},
            "frac_of_bf16_tensor_peak": achieved / peak,
            "algorithmic_flops_per_launch": flops}

    # ---- e2e through the public API (host step sequences -> fit epoch)
    e2e = None
    if rank == 0 and not args.no_e2e:
        seqs = as_seqs(steps, off, ctx)
        est2 = RecurrentAttentionTuner(batch_size=BATCH, loss="ranking", seed=0, epochs=0)
        est2.precision = "fp32"
        est2.fit(seqs[:2], y[:2])
        est2.continue_fit(seqs, y, epochs=1, learning_rate=1e-3)  # warm
        torch.cuda.synchronize()
        wall = []
        for _ in range(max(1, min(args.steps, 3))):
            t0 = time.perf_counter()
            est2.continue_fit(seqs, y, epochs=1, learning_rate=1e-3)
            torch.cuda.synchronize()
            wall.append(time.perf_counter() - t0)
        h2d = steps.size * 4 + off.size * 8 + ctx.size * 4 + y.size * 4 + n * 4 + n_steps * 16
        d2h = n * 4 + int(flat.numel()) * 4 + 4
        e2e = {"value": n / float(np.mean(wall)), "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "api": "RecurrentAttentionTuner.continue_fit(seqs, y, epochs=1)",
               "s_per_step": float(np.mean(wall))}

    # ---- secondary: bulk scoring and PCA throughput (configs 3 and 4 shapes)
    extra = {}
    if dist is not None and not args.no_extra:
        extra.update(sharded_extra(world, rank, dist, l2, stream, est, dims, flat))
    if rank == 0 and not args.no_extra:
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        est._set_host(est.__dict__["_host"])
        for _ in range(2):
            est._predict_programs(prog, dims, flat)
        flush_l2(l2)
        s0.record(stream)
        est._predict_programs(prog, dims, flat)
        s1.record(stream)
        torch.cuda.synchronize()
        sc_t = s0.elapsed_time(s1) / 1e3
        extra["scoring_programs_per_s"] = n / sc_t
        extra["scoring_tflops"] = float(np.sum(134656.0 * lens + 45568.0)) / sc_t / 1e12
        extra["scoring_fp32_path"] = ("tt_tuner_predict_f32tc: split-precision tcgen05 biLSTM "
                                      "(x_hi.w_hi + x_lo.w_hi + x_hi.w_lo) + fp32 CUDA-core attention")
        # where it sits (DESIGN 3.2b): the biLSTM's dense FLOPs run 3x on the
        # tensor cores (three tf32 chains), its cell issues 8 MUFU ops per
        # hidden unit and step; both against this box's peaks
        lstm_flops = float(np.sum(2.0 * 58880.0 * lens))  # 3 layers x 2 dirs, x and h GEMVs
        mufu_ops = float(np.sum(6.0 * 32 * 8 * lens))
        tf32_peak = 0.5 * float(peaks.get("bf16_tflops_sustained", 1400.0))
        extra["scoring_fp32_roofline"] = {
            "bound": "latency of the per-step chain (gates -> x -> cell -> h MMAs)",
            "tensor_tflops_tf32": 3.0 * lstm_flops / sc_t / 1e12,
            "frac_of_tf32_peak": 3.0 * lstm_flops / sc_t / 1e12 / tf32_peak,
            "mufu_ops_per_s": mufu_ops / sc_t,
            "frac_of_mufu_peak": mufu_ops / sc_t / 4.62e12,
            "peaks": f"tf32 = bf16_tflops_sustained / 2 = {tf32_peak:.0f} TFLOP/s (MEASURED_PEAKS.json); "
                     "MUFU 4.62e12 ops/s (profiles/r2_issue_peaks.json)"}
        # the strict CUDA-core fp32 kernel ("fp32_cuda", the round-1 default)
        est.precision = "fp32_cuda"
        est._predict_programs(prog, dims, flat)
        flush_l2(l2)
        s0.record(stream)
        est._predict_programs(prog, dims, flat)
        s1.record(stream)
        torch.cuda.synchronize()
        extra["scoring_fp32_cuda_programs_per_s"] = n / (s0.elapsed_time(s1) / 1e3)
        est.precision = "fp32"
        # the same scoring on the tensor cores (tcgen05 kind::tf32, "tf32" mode)
        est.precision = "tf32"
        for _ in range(2):
            est._predict_programs(prog, dims, flat)
        ts = []
        for _ in range(3):
            flush_l2(l2)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            est._predict_programs(prog, dims, flat)
            e1.record(stream)
            ts.append((e0, e1))
        torch.cuda.synchronize()
        tc_t = float(np.mean([a_.elapsed_time(b_) for a_, b_ in ts])) / 1e3
        est.precision = "fp32"
        extra["scoring_tc_tf32_programs_per_s"] = n / tc_t
        extra["scoring_tc_tf32_tflops"] = float(np.sum(134656.0 * lens + 45568.0)) / tc_t / 1e12
        from paper_2304_05430_b200 import metrics as gm

        pred = est._predict_programs(prog, dims, flat).double()
        toff = np.arange(0, n + 1, PER_TASK, dtype=np.int64)
        yt = torch.tensor(y, dtype=torch.float64, device="cuda")
        gm.pca_counts(yt, pred, toff)
        torch.cuda.synchronize()
        pts = []
        for _ in range(5):  # wall clock incl. the host-side plan and the D2H of the counts
            p0 = time.perf_counter()
            c = gm.pca_counts(yt, pred, toff)
            pts.append(time.perf_counter() - p0)
        pt = float(np.median(pts))
        pairs = N_TASKS * PER_TASK * (PER_TASK - 1) / 2
        extra["pca_pairs_per_s"] = pairs / pt
        extra["pca_mean"] = float(np.mean(c / (PER_TASK * (PER_TASK - 1) / 2)))
        extra.update(mlp_scoring(l2, stream, peaks))
        # large-batch variants of C2: one epoch at B = 256 / 1024
        for bb in (256, 1024):
            nsb = (n + bb - 1) // bb
            fl, mm, vv = flat.clone(), torch.zeros_like(flat), torch.zeros_like(flat)
            ts = []
            for k in range(2):
                pb = _device.to_dev(rng.permutation(n).astype(np.int32))
                cb = _device.to_dev(_bias_corrections(k * nsb, nsb))
                flush_l2(l2)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                est._launch_train(dims, fl, mm, vv, prog, yd, pb, bb, _lib.TT_MODE_TRAIN, 1e-3, cb, None)
                e1.record(stream)
                ts.append((e0, e1))
            torch.cuda.synchronize()
            extra[f"train_b{bb}_samples_per_s"] = n / (ts[-1][0].elapsed_time(ts[-1][1]) / 1e3)
        # search-time scoring latency through the public API (host sequences
        # in, float64 scores out): one SA step scores 1, one evolution
        # generation <= 32 candidates (search.py:319, :392-410)
        few = as_seqs(steps, off, ctx)[:32]
        for k_ in (1, 32):
            est.predict(few[:k_])
            w = []
            for _ in range(20):
                t0_ = time.perf_counter()
                est.predict(few[:k_])
                w.append(time.perf_counter() - t0_)
            extra[f"predict_latency_{k_}_us"] = float(np.median(w)) * 1e6
        extra.update(survey_configs(est, dims, flat, l2, stream, n_steps, prog, yd, rng))
        extra.update(mlp_training())
        extra.update(dp_exchange_cost())
        extra.update(search_throughput())
        extra.update(gbdt_fit_throughput())

    if rank == 0:
        cpu = None
        if not args.no_cpu:
            import refbench

            if refbench.available():
                cpu = refbench.reference_training(steps, off, ctx, y, n_sample=512, seconds=12.0)
                cpu["host"] = refbench.host_cores()
                if not args.no_extra:
                    # the scoring half of the metric: best-of-host reference scorers
                    cpu["scoring_best_of_host"] = sc = refbench.best_of_host_scoring(4.0)
                    if "scoring_programs_per_s" in extra:
                        extra["vs_best_of_host"] = {
                            "tuner_scoring_fp32": extra["scoring_programs_per_s"] / sc["tuner"]["value"],
                            "tuner_scoring_fp32_cuda": (extra["scoring_fp32_cuda_programs_per_s"]
                                                        / sc["tuner"]["value"]),
                            "tuner_scoring_tf32": extra["scoring_tc_tf32_programs_per_s"] / sc["tuner"]["value"],
                            "mlp_scoring_fp32": extra["mlp_fp32_rows_per_s"] / sc["mlp"]["value"],
                            "mlp_scoring_tf32": extra["mlp_tf32_rows_per_s"] / sc["mlp"]["value"],
                            "pca": extra["pca_pairs_per_s"] / sc["pca"]["value"],
                        }
            else:
                cpu = cpu_baseline(steps, off, ctx, y)
        line = {
            "metric": "rank-loss train samples/sec", "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_mean * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "attention tuner (3x biLSTM h32, 2 heads x 2 passes) rank-loss "
                                   "training, 64 tasks x 4096 programs, batch 16, Adam; 1 step = 1 epoch",
                       "global_batch": BATCH * world, "seq_len": int(lens.max()),
                       "parallelism": f"dp{world}" if world > 1 else "single",
                       "dp_exchange": dp_kind,
                       "l2": "flushed (256 MB write) between timed epochs"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            # one cooperative training launch per epoch per rank (fused DP
            # included); the NCCL fallback launches gradient + Adam per step
            "gpu_launches": args.steps if world == 1 or "fused" in dp_kind else 2 * n_steps * args.steps,
            "clocks": clocks.summary(int(os.environ.get("LOCAL_RANK", 0))),
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _selftest_launch(world, rank):
    """--selftest-launch: the launcher and the max-over-ranks plumbing without
    a GPU (gloo): every rank joins, contributes its rank, rank 0 prints."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    v = torch.tensor([float(rank)])
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    n = torch.tensor([1.0])
    dist.all_reduce(n)
    if rank == 0:
        print(json.dumps({"selftest": True, "n_gpus": world, "ranks_joined": int(n.item()),
                          "max_rank": int(v.item())}), flush=True)
    dist.destroy_process_group()


def _run(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.selftest_launch:
        _selftest_launch(world, rank)
    elif args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_b200(args, world, rank)


def _spawned(local_rank, args, world, port):
    os.environ.update({"RANK": str(local_rank), "LOCAL_RANK": str(local_rank), "WORLD_SIZE": str(world),
                       "LOCAL_WORLD_SIZE": str(world), "MASTER_ADDR": "127.0.0.1",
                       "MASTER_PORT": str(port)})
    _run(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--phase-batch", type=int, default=BATCH, help="minibatch of the --phases probe")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--profile", action="store_true", help="small dataset for ncu captures")
    ap.add_argument("--phases", action="store_true", help="print per-phase train-step timings")
    ap.add_argument("--selftest-launch", action="store_true",
                    help="exercise the N-rank launcher with gloo, no GPU work")
    args = ap.parse_args()
    if args.profile:
        args.no_cpu = args.no_e2e = True
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # not under torchrun: launch the N ranks ourselves (one process per
        # GPU, rendezvous on 127.0.0.1), same env contract as torchrun
        import socket

        import torch.multiprocessing as mp

        if not args.selftest_launch and args.impl == "b200":
            import torch

            have = torch.cuda.device_count()
            if have < args.gpus:
                raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        mp.spawn(_spawned, args=(args, args.gpus, port), nprocs=args.gpus, join=True)
        return
    _run(args)


if __name__ == "__main__":
    main()
