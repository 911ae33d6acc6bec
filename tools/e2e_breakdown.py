"""Host-side costs of one continue_fit epoch (bench's e2e) outside the kernel."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_05430_b200 import RecurrentAttentionTuner, _device  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms  # noqa: E402

steps, off, ctx, y, lens = bench.synth()
seqs = bench.as_seqs(steps, off, ctx)
est = RecurrentAttentionTuner(batch_size=16, loss="ranking", seed=0, epochs=0)
est.precision = "fp32"
est.fit(seqs[:2], y[:2])
est.continue_fit(seqs, y, epochs=1, learning_rate=1e-3)
dims = est._dims()


def tm(f, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


prog = DevicePrograms.from_sequences(seqs, "fp32", 6, 35)
print(f"from_sequences {tm(lambda: DevicePrograms.from_sequences(seqs, 'fp32', 6, 35)):.1f} ms")
print(f"y upload {tm(lambda: _device.to_dev(y, torch.float32)):.1f} ms")
print(f"permutation {tm(lambda: np.random.default_rng(0).permutation(len(y)).astype(np.int32)):.1f} ms")
from paper_2304_05430_b200.estimators import _bias_corrections  # noqa: E402
print(f"bias corrections {tm(lambda: _bias_corrections(0, 16384)):.1f} ms")
print(f"curve predict + rmse {tm(lambda: float(np.sqrt(np.mean((est._predict_programs(prog, dims).cpu().double().numpy() - y) ** 2)))):.1f} ms")
print(f"continue_fit total {tm(lambda: est.continue_fit(seqs, y, epochs=1, learning_rate=1e-3), reps=2):.1f} ms")
