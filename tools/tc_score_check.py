"""Quick numbers for the tcgen05 tuner scorer: error vs the oracle and
throughput vs the fp32 CUDA-core kernel at the bench's scale."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import bench
from oracle import tuner as otuner
from paper_2304_05430_b200 import RecurrentAttentionTuner
from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms

steps, off, ctx, y, lens = bench.synth()
n = len(y)
seqs = bench.as_seqs(steps, off, ctx)
m = RecurrentAttentionTuner(epochs=0, seed=0)
m.precision = "fp32"
m.fit(seqs[:4], y[:4])
dims = m._dims()
sub = seqs[:2000]
ref = otuner.predict(otuner.init_params(0), sub)
for prec in ("fp32", "tf32"):
    m.precision = prec
    got = m.predict(sub)
    d = np.abs(got - ref)
    print(f"{prec}: max|d| {d.max():.3e} mean|d| {d.mean():.3e}")
    prog = DevicePrograms(HostPrograms(steps, off, ctx), "fp32")
    flat = m._dev_params(dims)
    for _ in range(2):
        m._predict_programs(prog, dims, flat)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        m._predict_programs(prog, dims, flat)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3 / 1e3
    print(f"{prec}: {n / t / 1e6:.2f} M programs/s ({t * 1e3:.2f} ms for {n})")

import ctypes
from paper_2304_05430_b200 import _lib
buf = (ctypes.c_int64 * 32)()
_lib.load().tt_debug_tc_phase_times(buf, 32)
mk = list(buf)
cyc = lambda a, b: (mk[b] - mk[a])
print("tile:", " ".join(f"layer{l}={cyc(l, l + 1)}" for l in range(3)), f"attn-staging={cyc(3, 26)} attn={cyc(26, 20)} head={cyc(20, 21)} total={cyc(0, 21)} cycles")
print(f"layer1 step1: writeA={cyc(22, 23)} mma(wait)={cyc(23, 24)} epilogue={cyc(24, 25)} cycles")
print(f"attention: p0={cyc(26, 27)} pass0 q+r gemms={cyc(27, 28)} logits+softmax+u={cyc(28, 29)} rest={cyc(29, 20)}")
