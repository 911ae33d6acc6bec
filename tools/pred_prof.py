import sys; sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_2304_05430_b200 import RecurrentAttentionTuner
from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms
steps, off, ctx, y, lens = bench.synth(n_tasks=16, per_task=4096)
prog = DevicePrograms(HostPrograms(steps, off, ctx), "fp32")
est = RecurrentAttentionTuner(epochs=0, seed=0); est.precision = "fp32"; est._init_params()
dims = est._dims()
for _ in range(3): est._predict_programs(prog, dims)
torch.cuda.synchronize()
