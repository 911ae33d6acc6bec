"""Time the fp32 tuner scorer of a library variant (TT_LIB) on the bench's
262,144 programs; print programs/s and a checksum of the scores."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_05430_b200 import RecurrentAttentionTuner, _lib  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms  # noqa: E402

st, of, cx, y, ln = bench.synth(seed=0)
prog = DevicePrograms(HostPrograms(st, of, cx), "fp32")
est = RecurrentAttentionTuner(seed=0)
est._init_params()
est.precision = sys.argv[1] if len(sys.argv) > 1 else "fp32"
dims = est._dims()
flat = est._dev_params(dims)
for _ in range(2):
    out = est._predict_programs(prog, dims, flat)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = est._predict_programs(prog, dims, flat)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
o = out.cpu().numpy().astype(np.float64)
print(json.dumps({"lib": _lib.LIB_PATH, "programs_per_s": prog.n / float(np.median(ts)),
                  "checksum": float(o.sum()), "first": [float(v) for v in o[:3]]}))
