"""Per-step time of the generic training kernel (the fallback for programs
longer than the latency path admits / hidden != 32) vs the latency path."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib  # noqa: E402
from paper_2304_05430_b200.estimators import _bias_corrections  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms  # noqa: E402

for T_fix in (None, 24):
    steps, off, ctx, y, lens = bench.synth(n_tasks=2, per_task=4096)
    if T_fix:  # every program T_fix steps (beyond the latency path's limit)
        n = len(y)
        lens = np.full(n, T_fix)
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        steps = np.random.default_rng(0).normal(size=(int(off[-1]), 6))
    prog = DevicePrograms(HostPrograms(steps, off, ctx), "fp32")
    yd = _device.to_dev(y, torch.float32)
    est = RecurrentAttentionTuner(batch_size=16, loss="ranking", seed=0)
    est.precision = "fp32"
    est._init_params()
    dims = est._dims()
    n = prog.n
    ns = (n + 15) // 16
    for path in ((1, 2) if T_fix is None else (1,)):
        _lib.call("tt_tuner_train_set_path", path)
        flat = est._dev_params(dims).clone()
        m, v = torch.zeros_like(flat), torch.zeros_like(flat)
        perm = _device.to_dev(np.random.default_rng(1).permutation(n).astype(np.int32))
        corr = _device.to_dev(_bias_corrections(0, ns))
        est._launch_train(dims, flat, m, v, prog, yd, perm, 16, _lib.TT_MODE_TRAIN, 1e-3, corr, None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        est._launch_train(dims, flat, m, v, prog, yd, perm, 16, _lib.TT_MODE_TRAIN, 1e-3, corr, None)
        e1.record()
        torch.cuda.synchronize()
        name = {1: "generic", 2: "latency path"}[path]
        print(f"T {'hist' if T_fix is None else T_fix}: {name} {e0.elapsed_time(e1) * 1e3 / ns:.1f} us per step")
    _lib.call("tt_tuner_train_set_path", 0)
