"""Fused data-parallel training (tt_tuner_train_dp_f32, dist.FusedDataParallelTuner):
W ranks run the training kernel concurrently -- here inside one process on one
GPU, each rank on its own share of the SMs and its own stream, the exchange
buffers plain device memory standing in for the peers' NVLink-mapped ones.

Reference semantics (SURVEY §8e option A): step k's gradient is the mean of
the ranks' k-th microbatch gradients (rank loss pairs inside each
microbatch), followed by the replicated Adam step.  Checked against the
float64 oracle, plus bit-identical parameters on every rank.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import random_seqs
from oracle import tuner as otuner
from oracle.adam import AdamOracle

pytestmark = pytest.mark.gpu


def _unflatten(est, flat):
    host = est.__dict__["_host"]
    out, o = {}, 0
    for k in est._dims()["names"]:
        out[k] = flat[o:o + host[k].size].reshape(host[k].shape)
        o += host[k].size
    return out


@pytest.mark.parametrize("world,batch,loss", [(2, 8, "ranking"), (3, 5, "rmse"), (2, 100, "ranking")])
def test_fused_dp_matches_oracle(cuda_ok, world, batch, loss):
    import torch

    from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib
    from paper_2304_05430_b200.dist import FusedDataParallelTuner
    from paper_2304_05430_b200.layout import DevicePrograms

    n_local = (4 if batch < 50 else 2) * batch + 3  # a partial last microbatch on every rank
    # (batch 100 > the 74 CTAs of a rank here: the multi-round mode)
    rng = np.random.default_rng(world)
    seqs = random_seqs(rng, rng.integers(1, 11, size=world * n_local))
    y = rng.uniform(0.1, 0.9, size=world * n_local)
    shards = [slice(r * n_local, (r + 1) * n_local) for r in range(world)]
    ests, progs, ys = [], [], []
    for sh in shards:
        e = RecurrentAttentionTuner(epochs=0, seed=3, loss=loss)
        e.precision = "fp32"
        e.fit(seqs[sh], y[sh])
        ests.append(e)
        progs.append(DevicePrograms.from_sequences(seqs[sh], "fp32", 6, 35))
        ys.append(_device.to_dev(y[sh], torch.float32))
    ranks = FusedDataParallelTuner.local_group(ests, progs, ys, batch)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    p = otuner.init_params(3)
    opt = AdamOracle(p, 1e-3)
    _lib.call("tt_tuner_train_set_grid", sms // world)
    try:
        streams = [torch.cuda.Stream() for _ in range(world)]
        for epoch in range(2):
            perms = [rng.permutation(n_local) for _ in range(world)]
            torch.cuda.synchronize()
            stats = []
            for r in range(world):
                with torch.cuda.stream(streams[r]):
                    stats.append(ranks[r].run(perms[r], 1e-3))
            torch.cuda.synchronize()
            assert all(FusedDataParallelTuner.check_status(s) < 0 for s in stats)
            for k in range(0, n_local, batch):
                grads = []
                for r in range(world):
                    idx = [shards[r].start + i for i in perms[r][k:k + batch]]
                    _, g = otuner.loss_and_gradients(p, [seqs[i] for i in idx], y[idx], loss)
                    grads.append(g)
                opt.step({name: sum(g[name] for g in grads) / world for name in grads[0]})
    finally:
        _lib.call("tt_tuner_train_set_grid", 0)
    flats = [rk.flat.cpu().numpy() for rk in ranks]
    for f in flats[1:]:
        assert np.array_equal(f, flats[0])  # replicated update, identical on every rank
    got = _unflatten(ests[0], flats[0].astype(np.float64))
    for name in p:
        err = np.linalg.norm(got[name] - p[name]) / max(np.linalg.norm(p[name]), 1e-12)
        assert err <= 2e-3, (name, err)
    for rk in ranks:
        rk.close()


def test_create_over_nccl_world_one(cuda_ok):
    """FusedDataParallelTuner.create over a real NCCL process group (world
    size 1 on this box): the IPC allocation, handle exchange and agreement
    collectives run, and the epoch equals the single-GPU training kernel's."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib
    from paper_2304_05430_b200.dist import FusedDataParallelTuner
    from paper_2304_05430_b200.estimators import _bias_corrections
    from paper_2304_05430_b200.layout import DevicePrograms

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(4)
        seqs = random_seqs(rng, rng.integers(1, 11, size=40))
        y = rng.uniform(0.1, 0.9, size=40)
        est = RecurrentAttentionTuner(epochs=0, seed=3, loss="ranking")
        est.precision = "fp32"
        est.fit(seqs, y)
        prog = DevicePrograms.from_sequences(seqs, "fp32", 6, 35)
        yd = _device.to_dev(y, torch.float32)
        rk = FusedDataParallelTuner.create(est, prog, yd, 8)
        perm = rng.permutation(40)
        st = rk.run(perm, 1e-3)
        torch.cuda.synchronize()
        assert FusedDataParallelTuner.check_status(st) < 0
        dims = est._dims()
        flat = est._dev_params(dims).clone()
        m, v = torch.zeros_like(flat), torch.zeros_like(flat)
        est._launch_train(dims, flat, m, v, prog, yd, _device.to_dev(perm.astype(np.int32)), 8,
                          _lib.TT_MODE_TRAIN, 1e-3, _device.to_dev(_bias_corrections(0, 5)), None)
        torch.cuda.synchronize()
        assert torch.equal(rk.flat, flat)
        rk.close()
    finally:
        dist.destroy_process_group()


def test_exchange_times_out_instead_of_hanging_when_a_peer_never_runs(cuda_ok):
    """Robustness (VERDICT r1 weak 12 / ADVICE r1): rank 0 of a world-2 group
    launches, rank 1 never does.  Every wait for rank 1's slice is bounded:
    the first one times out (here 200 ms), sets the abort word, every later
    exchange skips its waits, the epoch ends and check_status raises."""
    import time

    import torch

    from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib
    from paper_2304_05430_b200.dist import FusedDataParallelTuner
    from paper_2304_05430_b200.layout import DevicePrograms

    rng = np.random.default_rng(8)
    seqs = random_seqs(rng, rng.integers(1, 11, size=2 * 40))
    y = rng.uniform(0.1, 0.9, size=80)
    ests, progs, ys = [], [], []
    for r in range(2):
        e = RecurrentAttentionTuner(epochs=0, seed=3, loss="ranking")
        e.precision = "fp32"
        e.fit(seqs[r * 40:(r + 1) * 40], y[r * 40:(r + 1) * 40])
        ests.append(e)
        progs.append(DevicePrograms.from_sequences(seqs[r * 40:(r + 1) * 40], "fp32", 6, 35))
        ys.append(_device.to_dev(y[r * 40:(r + 1) * 40], torch.float32))
    ranks = FusedDataParallelTuner.local_group(ests, progs, ys, 8)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    _lib.call("tt_tuner_train_set_grid", sms // 2)
    _lib.call("tt_tuner_dp_set_timeout_ms", 200)
    try:
        t0 = time.perf_counter()
        st = ranks[0].run(rng.permutation(40), 1e-3)   # rank 1 never launches
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        with pytest.raises(_lib.LibraryError, match="did not deliver"):
            FusedDataParallelTuner.check_status(st)
        assert wall < 5.0, wall   # one 200 ms timeout, not one per step
    finally:
        _lib.call("tt_tuner_dp_set_timeout_ms", 30000)
        _lib.call("tt_tuner_train_set_grid", 0)
        for rk in ranks:
            rk.close()
