"""Where the time of a small `predict` goes (search-time scoring latency)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_05430_b200 import RecurrentAttentionTuner  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms  # noqa: E402

steps, off, ctx, y, lens = bench.synth(n_tasks=1, per_task=256)
seqs = bench.as_seqs(steps, off, ctx)
est = RecurrentAttentionTuner(epochs=0, seed=0).fit(seqs[:2], y[:2])
est.precision = "fp32"
dims = est._dims()


def med(f, reps=200):
    for _ in range(10):
        f()
    w = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        w.append(time.perf_counter() - t0)
    return np.median(w) * 1e6


for k in (1, 32):
    sub = seqs[:k]
    prog = DevicePrograms.from_sequences(sub, "fp32", 6, 35)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    est._predict_programs(prog, dims)
    e0.record()
    est._predict_programs(prog, dims)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={k}: predict() {med(lambda: est.predict(sub)):.1f} us | pack+upload "
          f"{med(lambda: DevicePrograms.from_sequences(sub, 'fp32', 6, 35)):.1f} us | launch+sync "
          f"{med(lambda: est._predict_programs(prog, dims)):.1f} us | kernel {e0.elapsed_time(e1) * 1e3:.1f} us"
          f" | D2H {med(lambda: est._predict_programs(prog, dims).cpu()):.1f} us")
