"""Cost of the fused data-parallel exchange, measured on one GPU: W ranks run
concurrently on disjoint SM sets (W x 148/W CTAs) versus one rank alone on
the same number of SMs; the difference per step is what the in-kernel slice
exchange (stores to the peers' buffers, release flags, acquire waits,
rank-order sums) adds.  The transport here is the GPU's own memory; over
NVLink each hop adds the link latency."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib  # noqa: E402
from paper_2304_05430_b200.dist import FusedDataParallelTuner  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms  # noqa: E402

B = 16
sms = torch.cuda.get_device_properties(0).multi_processor_count
res = {}
for world, same in ((1, False), (-2, False), (2, True), (2, False)):
    indep = world < 0  # |world| independent single-rank runs, concurrently
    world = abs(world)
    ranks, ests = [], []
    for r in range(world):
        steps, off, ctx, y, lens = bench.synth(n_tasks=8, per_task=4096, seed=0 if same else r)
        prog = DevicePrograms(HostPrograms(steps, off, ctx), "fp32")
        e = RecurrentAttentionTuner(batch_size=B, loss="ranking", seed=0)
        e.precision = "fp32"
        e._init_params()
        ests.append((e, prog, _device.to_dev(y, torch.float32)))
    if indep:
        ranks = [FusedDataParallelTuner.local_group([a], [b], [c], B)[0] for a, b, c in ests]
    else:
        ranks = FusedDataParallelTuner.local_group([a for a, _, _ in ests], [b for _, b, _ in ests],
                                                   [c for _, _, c in ests], B)
    _lib.call("tt_tuner_train_set_grid", sms // 2)
    streams = [torch.cuda.Stream() for _ in range(world)]
    n = ests[0][1].n
    rng = np.random.default_rng(0)
    times = []
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                ranks[r].run(rng.permutation(n), 1e-3)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    _lib.call("tt_tuner_train_set_grid", 0)
    steps_per_epoch = (n + B - 1) // B
    us = min(times[1:]) / steps_per_epoch * 1e6
    key = (world, same, indep)
    res[key] = us
    what = "independent concurrent runs" if indep else f"{'identical' if same else 'different'} shards"
    print(f"world={world} ({what}) on {sms // 2} SMs per rank: {us:.2f} us per step")
    for rk in ranks:
        rk.close()
base = res[(2, False, True)]
print(f"exchange cost per step over two independent concurrent runs: {res[(2, True, False)] - base:.2f} us "
      f"(identical shards), {res[(2, False, False)] - base:.2f} us (different shards: + the ranks' skew)")
