"""Small invocations of every hot kernel, for compute-sanitizer
(memcheck / racecheck / synccheck), see tools/sanitize.sh:

  tuner_train_fast_kernel (latency path, B = 16, and multi-round B = 300 on
  a reduced grid), the fused data-parallel kernel (2 ranks on one GPU), the
  generic train kernel (hidden 4), tuner_predict (fp32 tensor-core
  split-precision incl. its bulk path and programs without steps, fp32_cuda,
  fp64) and the tcgen05 tf32 scorer, mlp predict (fp32 / tf32) and mlp train, PCA, top-k,
  pruning statistics and the GBDT kernels.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import random_seqs  # noqa: E402

from paper_2304_05430_b200 import (CostMLP, GradientBoostedTrees, RecurrentAttentionTuner,  # noqa: E402
                                   _lib, pca_counts)
from paper_2304_05430_b200 import metrics as gm  # noqa: E402
from paper_2304_05430_b200.dist import FusedDataParallelTuner  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms  # noqa: E402
from paper_2304_05430_b200.sampling import filter_stats  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(0)
seqs = random_seqs(rng, rng.integers(1, 11, size=64))
y = rng.uniform(0.1, 0.9, size=64)


def step(name):
    return which in ("all", name)


if step("train"):
    RecurrentAttentionTuner(epochs=1, batch_size=16, loss="ranking", seed=0).fit(seqs, y)
    RecurrentAttentionTuner(epochs=1, batch_size=8, hidden_size=4, recurrent_layers=2, seed=0).fit(seqs, y)
if step("train_multiround"):
    _lib.call("tt_tuner_train_set_grid", 32)
    try:
        s2 = random_seqs(rng, rng.integers(1, 11, size=100))
        RecurrentAttentionTuner(epochs=1, batch_size=50, loss="ranking", seed=0).fit(s2, rng.uniform(size=100))
    finally:
        _lib.call("tt_tuner_train_set_grid", 0)
if step("dp"):
    ests, progs, ys = [], [], []
    for r in range(2):
        e = RecurrentAttentionTuner(epochs=0, seed=3, loss="ranking").fit(seqs[r * 32:(r + 1) * 32],
                                                                         y[r * 32:(r + 1) * 32])
        e.precision = "fp32"
        ests.append(e)
        progs.append(DevicePrograms.from_sequences(seqs[r * 32:(r + 1) * 32], "fp32", 6, 35))
        ys.append(torch.tensor(y[r * 32:(r + 1) * 32], dtype=torch.float32, device="cuda"))
    ranks = FusedDataParallelTuner.local_group(ests, progs, ys, 8)
    _lib.call("tt_tuner_train_set_grid", 74)
    try:
        streams = [torch.cuda.Stream() for _ in ranks]
        st = []
        for rk, s in zip(ranks, streams):
            with torch.cuda.stream(s):
                st.append(rk.run(rng.permutation(32), 1e-3))
        torch.cuda.synchronize()
        assert all(FusedDataParallelTuner.check_status(x) < 0 for x in st)
    finally:
        _lib.call("tt_tuner_train_set_grid", 0)
        for rk in ranks:
            rk.close()
if step("predict"):
    m = RecurrentAttentionTuner(epochs=0, seed=1).fit(seqs, y)
    for prec in ("fp32", "fp32_cuda", "fp64", "tf32"):
        m.precision = prec
        m.predict(seqs * 5)
    # the fp32 tensor-core scorer's bulk path (length sort, thread-per-program
    # attention) and programs without steps
    from conftest import Seq  # noqa: E402

    m.precision = "fp32"
    m.predict(seqs * 320)
    m.predict([Seq(np.zeros((0, 6)), seqs[0].context)] * 200 + seqs)
if step("mlp"):
    X = rng.normal(size=(300, 164))
    mm = CostMLP(epochs=1, seed=0, loss="ranking").fit(X, rng.normal(size=300))
    for prec in ("fp32", "tf32"):
        mm.precision = prec
        mm.predict(X)
if step("metrics"):
    off = np.array([0, 40, 41, 300, 1000])
    yy = np.round(rng.uniform(size=1000), 2)
    ss = rng.normal(size=1000)
    pca_counts(yy, ss, off)
    gm.segmented_topk(yy, ss, off, 5)
    gm.ranking_grad_segments(yy[:64], ss[:64], np.array([0, 16, 64]))
    filter_stats(rng.integers(1, 1 << 30, size=1000), rng.lognormal(-9, 0.5, size=1000),
                 rng.uniform(size=1000) > 0.05, off, 0.1, 8)
if step("gbdt"):
    X = np.round(rng.normal(size=(500, 6)), 1)
    GradientBoostedTrees(num_trees=3, max_depth=5, min_samples_leaf=2).fit(X, rng.normal(size=500),
                                                                          eval_set=(X[:50], np.zeros(50)))
torch.cuda.synchronize()
print("sanitize workload ok:", which)
