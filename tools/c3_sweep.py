"""Config 3: bulk scoring of 1 M / 4 M / 16 M / 64 M programs on
one B200: fp32 (the default: split-precision tcgen05 LSTM + fp32 attention),
tf32 (tcgen05) and, up to 4 M, fp32_cuda (the CUDA-core kernel); T drawn
from the generator histogram (4..10, mean 7.1) and fixed T = 8.

Inputs are generated ON THE DEVICE (torch, seeded) in the CSR layout the
kernels consume, so a 64 M-program sweep does not spend minutes in host
numpy; device time per launch with CUDA events (L2 flushed before each).
Prints one JSON line per (N, T mode, precision).

    python tools/c3_sweep.py [--sizes 1,4,16,64]
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2304_05430_b200 import RecurrentAttentionTuner  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms  # noqa: E402

T_HIST = {4: 35, 5: 196, 6: 457, 7: 516, 8: 469, 9: 291, 10: 46}


class _Dev(DevicePrograms):
    def __init__(self, steps, offsets, ctx, max_steps):  # noqa: D401 - device-built CSR
        self.precision = "fp32"
        self.steps, self.offsets, self.ctx = steps, offsets, ctx
        self.n = offsets.numel() - 1
        self.d0, self.C = 6, 35
        self.max_steps = max_steps
        self.host_offsets = None


def make(n, fixed_t, g):
    if fixed_t:
        lens = torch.full((n,), fixed_t, dtype=torch.int64, device="cuda")
    else:
        p = torch.tensor(list(T_HIST.values()), dtype=torch.float64, device="cuda")
        idx = torch.multinomial(p / p.sum(), n, replacement=True, generator=g)
        lens = torch.tensor(list(T_HIST), device="cuda")[idx]
    off = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    torch.cumsum(lens, 0, out=off[1:])
    rows = int(off[-1].item())
    steps = torch.zeros(rows, 6, device="cuda")
    kind = torch.randint(0, 4, (rows,), device="cuda", generator=g)
    steps[torch.arange(rows, device="cuda"), kind] = 1.0
    steps[:, 4] = torch.randint(0, 6, (rows,), device="cuda", generator=g).float()
    steps[:, 5] = torch.randint(-1, 3, (rows,), device="cuda", generator=g).float()
    ctx = torch.randn(n, 35, device="cuda", generator=g)
    return _Dev(steps.reshape(-1), off, ctx.reshape(-1), int(lens.max().item())), lens


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1,4,16,64")
    args = ap.parse_args()
    est = RecurrentAttentionTuner(seed=0)
    est._init_params()
    dims = est._dims()
    l2 = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    for m in [int(x) for x in args.sizes.split(",")]:
        n = m * 1024 * 1024
        for fixed in (0, 8):
            prog, lens = make(n, fixed, g)
            flops = float((134656.0 * lens.double() + 45568.0).sum().item())
            for prec in ("fp32", "tf32") + (("fp32_cuda",) if m <= 4 else ()):
                est.precision = prec
                flat = est._dev_params(dims)
                est._predict_programs(prog, dims, flat)
                ts = []
                for _ in range(3):
                    l2.fill_(1)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    out = est._predict_programs(prog, dims, flat)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / 1e3)
                t = float(np.median(ts))
                ok = bool(torch.isfinite(out).all().item() and ((out > 0) & (out < 1)).all().item())
                print(json.dumps({"programs": n, "T": "hist(4..10)" if not fixed else fixed, "precision": prec,
                                  "programs_per_s": n / t, "tflops": flops / t / 1e12, "s": t,
                                  "scores_in_(0,1)": ok}), flush=True)
            del prog, lens
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
