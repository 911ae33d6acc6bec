"""MLP tcgen05 scoring throughput at F=164 (the bench's extra)."""
import sys
sys.path.insert(0, ".")
import json
import torch
import bench

peaks = json.load(open("MEASURED_PEAKS.json")) if __import__("os").path.exists("MEASURED_PEAKS.json") else {}
l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
print(bench.mlp_scoring(l2, torch.cuda.current_stream(), peaks))

# error of the tf32 path vs float64 on a slice
import numpy as np
from paper_2304_05430_b200 import CostMLP
from oracle import mlp as omlp
rng = np.random.default_rng(0)
X = rng.normal(size=(4096, 164))
m = CostMLP(epochs=0, seed=0)
m.precision = "tf32"
m.fit(X[:64], rng.uniform(size=64))
got = m.predict(X)
m.precision = "fp64"
want = m.predict(X)
d = np.abs(got - want)
print("tf32 vs fp64: max", d.max(), "mean", d.mean())
