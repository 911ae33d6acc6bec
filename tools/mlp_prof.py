"""One launch of each CostMLP scorer at 4 M rows x F = 164 (for ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2304_05430_b200 import CostMLP, _device, _lib  # noqa: E402

n, F = 4 * 1024 * 1024, 164
X = torch.randn(n, F, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
est = CostMLP(epochs=0, seed=0)
est._init_params(F)
flat = est._device_flat(list(est.NAMES))
y = torch.empty(n, device="cuda")
which = sys.argv[1:] or ["tt_mlp_predict_f32tc", "tt_mlp_predict_tf32"]
for fn in which:
    for _ in range(2):
        _lib.call(fn, flat.data_ptr(), X.data_ptr(), n, F, y.data_ptr(), _device.stream_ptr())
torch.cuda.synchronize()
print("ok")
