"""Where the time of a small `predict` goes (search-time scoring latency)."""
import cProfile
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_05430_b200 import RecurrentAttentionTuner  # noqa: E402

steps, off, ctx, y, lens = bench.synth(n_tasks=1, per_task=256)
seqs = bench.as_seqs(steps, off, ctx)
est = RecurrentAttentionTuner(epochs=0, seed=0).fit(seqs[:2], y[:2])
est.precision = "fp32"
for k in (1, 32):
    for _ in range(20):
        est.predict(seqs[:k])
    w = []
    for _ in range(200):
        t0 = time.perf_counter()
        est.predict(seqs[:k])
        w.append(time.perf_counter() - t0)
    print(f"predict({k}): median {np.median(w) * 1e6:.1f} us, min {np.min(w) * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    est.predict(seqs[:1])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
