"""CostMLP training throughput: device time of one epoch (one launch) at the
reference's minibatch of 16, and fit() wall time including host work."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2304_05430_b200 import CostMLP, _device, _lib  # noqa: E402
from paper_2304_05430_b200.estimators import _bias_corrections  # noqa: E402

rng = np.random.default_rng(0)
for F, n in ((164, 65536), (47, 65536)):
    X = rng.normal(size=(n, F))
    y = rng.uniform(0.1, 0.9, size=n)
    m = CostMLP(epochs=1, batch_size=16, loss="ranking", seed=0)
    m.precision = "fp32"
    m.fit(X[:64], y[:64])
    t = time.perf_counter()
    m.fit(X, y)
    wall = time.perf_counter() - t
    flat = m._device_flat(list(m.NAMES)).clone()
    mm, vv = torch.zeros_like(flat), torch.zeros_like(flat)
    Xd = _device.to_dev(X.ravel(), torch.float32)
    yd = _device.to_dev(y, torch.float32)
    order = _device.to_dev(rng.permutation(n).astype(np.int32))
    steps = (n + 15) // 16
    corr = _device.to_dev(_bias_corrections(0, steps))
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m._launch_train(flat, mm, vv, Xd, yd, F, order, 16, _lib.TT_MODE_TRAIN, 1e-3, corr)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    dev = min(ts)
    print(f"F={F}: device {n / dev:,.0f} samples/s ({dev / steps * 1e6:.2f} us per Adam step); "
          f"fit() wall {n / wall:,.0f} samples/s")

# per-phase clock64 marks of minibatch 64 of the last launch (1965 MHz)
import ctypes  # noqa: E402

buf = (ctypes.c_int64 * 7)()
_lib.load().tt_debug_mlp_phase_times(buf, 7)
mk = list(buf)
names = ["stage+fwd", "out", "loss", "D2/D1", "W tiles+Adam", "bias/W3+Adam"]
print("phases (us):", ", ".join(f"{nm}={(mk[i + 1] - mk[i]) / 1965.0:.2f}" for i, nm in enumerate(names)))
