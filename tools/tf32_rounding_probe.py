"""Does tcgen05 kind::tf32 truncate or round its fp32 operands?  (Decides
how the split-precision "3xTF32" scorer forms its hi/lo halves.)

Runs the tf32 CostMLP scorer (A = X from shared memory) on rows whose first
feature is 1 + d for d below tf32 resolution (2^-10), with W1 = e_0 e_0^T,
b = 0, W2 = I, W3 = e_0: the score is a monotone function of the tensor
core's view of x.  Truncation maps every d < 2^-10 to 1.0 (equal scores);
round-to-nearest maps d >= 2^-11 to 1 + 2^-10."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2304_05430_b200 import _device, _lib  # noqa: E402

F = 32
prm = np.zeros(F * 64 + 64 + 64 * 64 + 64 + 64 + 1, dtype=np.float32)
W1 = np.zeros((F, 64), np.float32)
W1[0, 0] = 1.0
o = 0
prm[o:o + F * 64] = W1.ravel(); o += F * 64 + 64
prm[o:o + 64 * 64] = np.eye(64, dtype=np.float32).ravel(); o += 64 * 64 + 64
prm[o] = 1.0  # W3[0]
ds = [0.0, 2.0**-13, 2.0**-12, 2.0**-11 - 2.0**-20, 2.0**-11, 2.0**-11 + 2.0**-13, 2.0**-10 - 2.0**-20, 2.0**-10]
X = np.zeros((128, F), np.float32)
for i, d in enumerate(ds):
    X[i, 0] = np.float32(1.0 + d)
dp = _device.to_dev(prm)
dx = _device.to_dev(X)
out = torch.empty(128, device="cuda")
_lib.call("tt_mlp_predict_tf32", dp.data_ptr(), dx.data_ptr(), 128, F, out.data_ptr(), _device.stream_ptr())
s = out.cpu().numpy()[: len(ds)]
for d, v in zip(ds, s):
    print(f"d = {d:.3e}  score = {v:.9f}  same_as_d0 = {v == s[0]}")
print("VERDICT:", "truncate" if s[5] == s[0] else ("round" if s[5] == s[-1] else "other"))
