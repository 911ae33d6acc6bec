"""N > 1 host logic on CPU: world_size-2 gloo process groups (127.0.0.1).

The per-rank compute is the oracle here (these tests run without a GPU); the
sharding, the data-parallel gradient all-reduce (SURVEY §8e option A) and the
exact PCA count reduction are the production code paths of
paper_2304_05430_b200.dist.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import random_seqs


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _dp_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import tuner as otuner
    from paper_2304_05430_b200 import dist as tdist

    _init(rank, world, port)
    rng = np.random.default_rng(0)
    seqs = random_seqs(rng, rng.integers(1, 6, size=37))
    y = rng.uniform(0.1, 0.9, size=37)
    p = otuner.init_params(1, layers=1, hidden=4)
    names = list(p)
    perm = np.random.default_rng(5).permutation(37)
    B = 4
    steps = tdist.dp_steps(37, B, world)
    grads = []
    for k in range(steps):
        mb = tdist.dp_microbatch(perm, k, B, rank, world)
        if len(mb):
            _, g = otuner.loss_and_gradients(p, [seqs[i] for i in mb], y[mb], "ranking")
            flat = torch.tensor(np.concatenate([g[n].ravel() for n in names]))
        else:
            flat = torch.zeros(sum(p[n].size for n in names), dtype=torch.float64)
        tdist.mean_microbatch_gradient(flat, len(mb))
        grads.append(flat.numpy().copy())
    out[rank] = np.stack(grads)
    dist.destroy_process_group()


def test_dp_gradient_allreduce_equals_mean_of_microbatch_gradients():
    from oracle import tuner as otuner
    from paper_2304_05430_b200 import dist as tdist

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_dp_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert np.array_equal(out[0], out[1])  # every replica applies the same update
    rng = np.random.default_rng(0)
    seqs = random_seqs(rng, rng.integers(1, 6, size=37))
    y = rng.uniform(0.1, 0.9, size=37)
    p = otuner.init_params(1, layers=1, hidden=4)
    names = list(p)
    perm = np.random.default_rng(5).permutation(37)
    for k in range(tdist.dp_steps(37, 4, world)):
        parts = []
        for r in range(world):
            mb = tdist.dp_microbatch(perm, k, 4, r, world)
            if len(mb):
                _, g = otuner.loss_and_gradients(p, [seqs[i] for i in mb], y[mb], "ranking")
                parts.append(np.concatenate([g[n].ravel() for n in names]))
        np.testing.assert_allclose(out[0][k], np.mean(parts, axis=0), rtol=1e-12, atol=1e-15)


def _pca_worker(rank, world, port, sizes, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import metrics as om
    from paper_2304_05430_b200 import dist as tdist

    _init(rank, world, port)
    rng = np.random.default_rng(9)
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    off[1:] = np.cumsum(sizes)
    y = np.round(rng.normal(size=off[-1]), 1)
    s = np.round(rng.normal(size=off[-1]), 1)
    mine = tdist.lpt_assign(sizes, world)[rank]
    local = {t: om.pca_counts(y[off[t]:off[t + 1]], s[off[t]:off[t + 1]])[0]
             for t in mine if sizes[t] >= 2}
    out[rank] = tdist.gather_counts(local, len(sizes))
    dist.destroy_process_group()


def test_pca_counts_sharded_by_task_reduce_exactly():
    from oracle import metrics as om

    sizes = [50, 3, 120, 1, 77, 64, 2, 200, 9]
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_pca_worker, args=(world, _free_port(), sizes, out), nprocs=world, join=True)
    rng = np.random.default_rng(9)
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    off[1:] = np.cumsum(sizes)
    y = np.round(rng.normal(size=off[-1]), 1)
    s = np.round(rng.normal(size=off[-1]), 1)
    want = [om.pca_counts(y[off[t]:off[t + 1]], s[off[t]:off[t + 1]])[0] if sizes[t] >= 2 else 0
            for t in range(len(sizes))]
    assert list(out[0]) == want and list(out[1]) == want


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharding_helpers_partition_everything(world):
    from paper_2304_05430_b200 import dist as tdist

    rng = np.random.default_rng(world)
    lens = rng.integers(1, 11, size=1001)
    off = np.zeros(1002, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    ranges = tdist.shard_by_rows(off, world)
    assert ranges[0][0] == 0 and ranges[-1][1] == 1001
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    rows = [off[b] - off[a] for a, b in ranges]
    assert max(rows) - min(rows) <= 2 * lens.max()
    parts = tdist.lpt_assign(rng.integers(1, 100, size=57), world)
    assert sorted(t for p in parts for t in p) == list(range(57))
    perm = rng.permutation(103)
    seen = np.concatenate([tdist.dp_microbatch(perm, k, 4, r, world)
                           for k in range(tdist.dp_steps(103, 4, world)) for r in range(world)])
    assert np.array_equal(seen, perm)


def _handles_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2304_05430_b200 import dist as tdist

    _init(rank, world, port)
    out[rank] = tdist.exchange_handles(bytes([rank]) * 64)
    dist.destroy_process_group()


def test_ipc_handle_exchange_is_rank_ordered():
    """FusedDataParallelTuner.create's wiring: every rank receives every
    rank's exchange-buffer handle, in rank order (index = peer rank)."""
    world = 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_handles_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    want = [bytes([r]) * 64 for r in range(world)]
    assert all(list(out[r]) == want for r in range(world))


def test_dp_buffer_size_covers_every_slot():
    """tt_tuner_dp_buffer_bytes = flags (padded) + 2 parities x jobs x world
    x slice, slice >= the widest job slice (host-only entry point)."""
    from paper_2304_05430_b200 import _lib

    lib = _lib.load()
    one = lib.tt_tuner_dp_buffer_bytes(3, 32, 6, 35, 1)
    two = lib.tt_tuner_dp_buffer_bytes(3, 32, 6, 35, 2)
    assert one > 0 and two > one
    assert lib.tt_tuner_dp_buffer_bytes(3, 16, 6, 35, 2) == 0  # fused path is hidden-32 only
    wide = lib.tt_tuner_dp_buffer_bytes(3, 32, 164, 35, 2)
    assert wide > two  # wider layer-0 slices


def _unequal_worker(rank, world, port, out):
    """Shards of 37 and 20 samples: both ranks must loop to the longer
    shard's step count (DataParallelTunerEpoch deadlocked)."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2304_05430_b200 import dist as tdist

    _init(rank, world, port)
    n_local, B = (37, 20)[rank], 4
    steps = tdist.global_max_int((n_local + B - 1) // B)
    sums = []
    for k in range(steps):
        cnt = max(0, min(B, n_local - k * B))
        g = torch.full((3,), float(cnt), dtype=torch.float64)
        tdist.mean_microbatch_gradient(g, cnt)
        sums.append(float(g[0]))
    out[rank] = (steps, sums)
    dist.destroy_process_group()


def test_dp_unequal_local_shards_take_the_same_number_of_collectives():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_unequal_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] == out[1]
    steps, sums = out[0]
    assert steps == 10
    # steps 0-4: both ranks contribute 4; steps 5-8: only rank 0 (4); step 9: rank 0's 1
    assert sums == [4.0] * 9 + [1.0]


def _agree_worker(rank, world, port, pre, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2304_05430_b200 import _lib
    from paper_2304_05430_b200 import dist as tdist

    _init(rank, world, port)
    r = object.__new__(tdist.FusedDataParallelTuner)
    r.group = dist.group.WORLD
    try:
        r._agree(tuple(pre[rank]))
        out[rank] = "ok"
    except _lib.LibraryError as exc:
        out[rank] = "raised: " + str(exc)
    dist.destroy_process_group()


@pytest.mark.parametrize("pre,ok", [
    ([(10, 0, 1), (10, 0, 1)], True),
    ([(10, 0, 1), (9, 0, 1)], False),    # a shorter shard
    ([(10, 5, 1), (10, 0, 1)], False),   # diverged global step base
    ([(10, 0, 1), (10, 0, 0)], False),   # one rank holds a program too long for the kernel
])
def test_fused_dp_preconditions_agree_or_raise_on_every_rank(pre, ok):
    """a rank that cannot launch (or launches fewer steps) must not
    leave its peers spinning in the exchange -- all ranks raise together."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_agree_worker, args=(world, _free_port(), pre, out), nprocs=world, join=True)
    if ok:
        assert out[0] == out[1] == "ok"
    else:
        assert out[0].startswith("raised") and out[1].startswith("raised")


def _sharded_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import metrics as om
    from oracle import tuner as otuner
    from paper_2304_05430_b200 import dist as tdist

    _init(rank, world, port)
    rng = np.random.default_rng(3)
    seqs = random_seqs(rng, rng.integers(1, 9, size=41))
    p = otuner.init_params(2, layers=1, hidden=4)
    calls = []

    def pred(_est, s):
        calls.append(len(s))
        return otuner.predict(p, s)

    scores = tdist.sharded_predict(None, seqs, predict_fn=pred)
    sizes = [50, 3, 120, 1, 77, 64, 2, 200, 9, 0]
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    off[1:] = np.cumsum(sizes)
    y = np.round(rng.normal(size=off[-1]), 1)
    s = np.round(rng.normal(size=off[-1]), 1)

    def cnt(yy, ss, sub):
        return np.array([om.pca_counts(yy[sub[i]:sub[i + 1]], ss[sub[i]:sub[i + 1]])[0]
                         for i in range(len(sub) - 1)], dtype=np.int64)

    counts = tdist.sharded_pca_counts(y, s, off, count_fn=cnt)
    out[rank] = (scores, calls, counts)
    dist.destroy_process_group()


def test_sharded_predict_and_pca_equal_unsharded():
    """e1/e2 entry points (dist.sharded_predict / sharded_pca_counts): each
    rank computes only its shard, the host gather / one int64 all-reduce
    reassembles exactly the unsharded result on every rank."""
    from oracle import metrics as om
    from oracle import tuner as otuner

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sharded_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    rng = np.random.default_rng(3)
    seqs = random_seqs(rng, rng.integers(1, 9, size=41))
    want = otuner.predict(otuner.init_params(2, layers=1, hidden=4), seqs)
    sizes = [50, 3, 120, 1, 77, 64, 2, 200, 9, 0]
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    off[1:] = np.cumsum(sizes)
    y = np.round(rng.normal(size=off[-1]), 1)
    s = np.round(rng.normal(size=off[-1]), 1)
    wc = [om.pca_counts(y[off[t]:off[t + 1]], s[off[t]:off[t + 1]])[0] if sizes[t] >= 2 else 0
          for t in range(len(sizes))]
    for r in range(world):
        scores, calls, counts = out[r]
        np.testing.assert_allclose(scores, want, rtol=1e-12)
        assert len(calls) == 1 and 0 < calls[0] < 41  # each rank scored only its shard
        assert list(counts) == wc
    assert out[0][1][0] + out[1][1][0] == 41
