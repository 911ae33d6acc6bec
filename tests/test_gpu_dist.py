"""Multi-rank entry points on the GPU, runnable on one B200:

* dist.sharded_predict / sharded_pca_counts with two ranks (two processes on
  cuda:0, gloo for the host plumbing) running the real kernels on their
  shards, against the unsharded kernels -- bit-identical;
* the same over a real NCCL process group of world size 1;
* DataParallelTunerEpoch (gradient launch + NCCL all-reduce + standalone
  Adam launch per step) over NCCL world 1 against the float64 oracle;
* the standalone fused Adam kernels (tt_adam_step_f32/_f64) against the
  reference's golden Adam trajectory (tests/golden/adam.npz).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import golden, random_seqs

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    rng = np.random.default_rng(12)
    seqs = random_seqs(rng, rng.integers(1, 13, size=3000))
    sizes = np.array([700, 1, 513, 64, 2, 1200, 0, 520])
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    off[1:] = np.cumsum(sizes)
    y = np.round(rng.uniform(size=off[-1]), 2)
    return seqs, y, off


def _sharded_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    from paper_2304_05430_b200 import RecurrentAttentionTuner
    from paper_2304_05430_b200 import dist as tdist

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seqs, y, off = _data()
    est = RecurrentAttentionTuner(epochs=0, seed=5).fit(seqs[:4], y[:4])
    lo, hi, local = tdist.sharded_predict(est, seqs, gather=False)
    full = tdist.sharded_predict(est, seqs)
    counts = tdist.sharded_pca_counts(y, full, off)
    out[rank] = (lo, hi, local, full, counts)
    dist.destroy_process_group()


def test_sharded_scoring_and_pca_two_ranks_on_one_gpu(cuda_ok):
    import torch.multiprocessing as mp

    from paper_2304_05430_b200 import RecurrentAttentionTuner, pca_counts

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sharded_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    seqs, y, off = _data()
    est = RecurrentAttentionTuner(epochs=0, seed=5).fit(seqs[:4], y[:4])
    want = est.predict(seqs)
    want_c = pca_counts(y, want, off)
    (lo0, hi0, l0, f0, c0), (lo1, hi1, l1, f1, c1) = out[0], out[1]
    assert lo0 == 0 and hi0 == lo1 and hi1 == len(seqs) and 0 < hi0 < len(seqs)
    # per-program arithmetic is independent of the batch: bit-identical
    np.testing.assert_array_equal(np.concatenate([l0, l1]), want)
    np.testing.assert_array_equal(f0, want)
    np.testing.assert_array_equal(f1, want)
    np.testing.assert_array_equal(c0, want_c)
    np.testing.assert_array_equal(c1, want_c)


def _nccl_world_one():
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    return dist


def test_sharded_entry_points_over_nccl_world_one(cuda_ok):
    from paper_2304_05430_b200 import RecurrentAttentionTuner, pca_counts
    from paper_2304_05430_b200 import dist as tdist

    dist = _nccl_world_one()
    try:
        seqs, y, off = _data()
        est = RecurrentAttentionTuner(epochs=0, seed=5).fit(seqs[:4], y[:4])
        got = tdist.sharded_predict(est, seqs)
        np.testing.assert_array_equal(got, est.predict(seqs))
        np.testing.assert_array_equal(tdist.sharded_pca_counts(y, got, off), pca_counts(y, got, off))
        pca = tdist.sharded_segmented_pca(y, got, off)
        assert np.isnan(pca[1]) and np.isnan(pca[6]) and np.all((pca[[0, 2, 3]] >= 0) & (pca[[0, 2, 3]] <= 1))
    finally:
        dist.destroy_process_group()


def test_nccl_dataparallel_epoch_matches_oracle(cuda_ok):
    """The NCCL fallback DP path (ADVICE/VERDICT r1: never ran with GPU
    kernels): fp64 build, world 1 (the all-reduce is the identity), two
    epochs over a local shard against the float64 oracle's Adam loop."""
    import torch

    from oracle import tuner as otuner
    from oracle.adam import AdamOracle
    from paper_2304_05430_b200 import RecurrentAttentionTuner, _device
    from paper_2304_05430_b200.dist import DataParallelTunerEpoch
    from paper_2304_05430_b200.layout import DevicePrograms

    dist = _nccl_world_one()
    try:
        rng = np.random.default_rng(2)
        seqs = random_seqs(rng, rng.integers(1, 8, size=27))
        y = rng.uniform(0.1, 0.9, size=27)
        est = RecurrentAttentionTuner(epochs=0, seed=4, hidden_size=4, recurrent_layers=2, loss="ranking")
        est.precision = "fp64"
        est.fit(seqs, y)
        prog = DevicePrograms.from_sequences(seqs, "fp64", 6, 35)
        dp = DataParallelTunerEpoch(est, prog, _device.to_dev(y, torch.float64), 8)
        p = otuner.init_params(4, layers=2, hidden=4)
        opt = AdamOracle(p, 1e-3)
        for _ in range(2):
            perm = rng.permutation(27)
            assert dp.run(perm, 1e-3, local_shard=True) == 4
            for k in range(0, 27, 8):
                b = perm[k:k + 8]
                _, g = otuner.loss_and_gradients(p, [seqs[i] for i in b], y[b], "ranking")
                opt.step(g)
        torch.cuda.synchronize()
        flat = dp.flat.cpu().numpy()
        o = 0
        for k in est._dims()["names"]:
            n = p[k].size
            np.testing.assert_allclose(flat[o:o + n].reshape(p[k].shape), p[k], rtol=1e-8, atol=1e-12,
                                       err_msg=k)
            o += n
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype,fn,rtol", [("float64", "tt_adam_step_f64", 0.0),
                                           ("float32", "tt_adam_step_f32", 2e-6)])
def test_standalone_adam_matches_reference_golden(cuda_ok, dtype, fn, rtol):
    """K8 standalone (optim.py:33-46): 3 steps of the reference's Adam with a
    tensor frozen at step 2 (absent from that step's grads -> mask 0, the
    shared step counter still advances), golden from the reference itself.
    fp64 is bit-exact (IEEE div/sqrt, no FMA contraction of the update)."""
    import torch

    from paper_2304_05430_b200 import _device, _lib

    g = golden("adam.npz")
    names = ("a", "b", "c")
    sizes = [g["init_" + k].size for k in names]
    tdt = getattr(torch, dtype)
    p = _device.to_dev(np.concatenate([g["init_" + k].ravel() for k in names]), tdt)
    m, v = torch.zeros_like(p), torch.zeros_like(p)
    for t in range(3):
        present = [f"g{t}_{k}" in g for k in names]
        grad = np.concatenate([g[f"g{t}_{k}"].ravel() if ok else np.zeros(s)
                               for k, ok, s in zip(names, present, sizes)])
        mask = np.concatenate([np.full(s, ok, dtype=np.uint8) for ok, s in zip(present, sizes)])
        gd, md = _device.to_dev(grad, tdt), _device.to_dev(mask)
        c1, c2 = 1.0 - 0.9 ** (t + 1), 1.0 - 0.999 ** (t + 1)
        _lib.call(fn, p.data_ptr(), gd.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel(), md.data_ptr(),
                  3e-3, 0.9, 0.999, 1e-8, c1, c2, _device.stream_ptr())
    got = p.cpu().double().numpy()
    want = np.concatenate([g["final_" + k].ravel() for k in names])
    if rtol == 0.0:
        np.testing.assert_array_equal(got, want)
    else:
        np.testing.assert_allclose(got, want, rtol=rtol)
