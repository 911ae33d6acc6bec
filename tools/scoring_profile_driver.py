"""One call of every scoring kernel at the bench's sizes, for a single
`ncu --set full` capture (tools/gpu_round.sh): tuner fp32 (tensor-core
default), fp32_cuda and tf32 on the bench's 262,144 programs; CostMLP fp32 /
tf32 / fp32_cuda on 4 M rows x 164; PCA counts over 64 tasks x 4096; GBDT
predict on 262,144 rows x 164.

    ncu --set full -k regex:'...' python tools/scoring_profile_driver.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_05430_b200 import CostMLP, GradientBoostedTrees, RecurrentAttentionTuner, _lib  # noqa: E402
from paper_2304_05430_b200 import metrics as gm  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms  # noqa: E402


def main():
    st, of, cx, y, ln = bench.synth(seed=0)
    prog = DevicePrograms(HostPrograms(st, of, cx), "fp32")
    est = RecurrentAttentionTuner(seed=0)
    est._init_params()
    dims = est._dims()
    flat = est._dev_params(dims)
    for prec in ("fp32", "fp32_cuda", "tf32"):
        est.precision = prec
        pred = est._predict_programs(prog, dims, flat)
    torch.cuda.synchronize()
    n, F = 4 * 1024 * 1024, 164
    X = torch.randn(n, F, device="cuda")
    mlp = CostMLP(epochs=0, seed=0)
    mlp._init_params(F)
    out = torch.empty(n, device="cuda")
    for prec, fn in (("fp32", "tt_mlp_predict_f32tc"), ("tf32", "tt_mlp_predict_tf32"),
                     ("fp32_cuda", "tt_mlp_predict_f32")):
        mlp.precision = prec
        fl = mlp._device_flat(list(mlp.NAMES))
        _lib.call(fn, fl.data_ptr(), X.data_ptr(), n, F, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    toff = np.arange(0, prog.n + 1, bench.PER_TASK, dtype=np.int64)
    yt = torch.tensor(y, dtype=torch.float64, device="cuda")
    gm.pca_counts(yt, pred.double(), toff)
    rng = np.random.default_rng(0)
    Xg = rng.normal(size=(4096, F))
    g = GradientBoostedTrees(num_trees=4, max_depth=6).fit(Xg, rng.uniform(size=4096))
    g.predict(rng.normal(size=(262144, F)))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
