"""Multi-GPU plumbing: one process per GPU, torch.distributed
(NCCL over NVLink on the box, gloo in CPU tests).

* scoring: programs are sharded into contiguous ranges of ~equal step-row
  count -- no collective on the data path (weak scaling);
* PCA: tasks are assigned by LPT on n_t^2 (the pair work); per-task
  (correct, total) are exact int64, so the final gather is order independent;
* training: data parallel.  Global minibatch k of size W*B is
  perm[k*W*B : (k+1)*W*B]; rank r takes its B-slice as the reference's
  minibatch (pairs of the rank loss stay inside it, SURVEY §8e option A) and
  the step gradient is the mean of the non-empty microbatch gradients,
  formed by one all-reduce before the (replicated) fused Adam update
  (DataParallelTunerEpoch, any kernel), or -- the B200 path --
  FusedDataParallelTuner: one training launch per epoch per rank whose
  gradient jobs exchange their slices with the peers through NVLink peer
  memory (tt_tuner_train_dp_f32), no separate collective or Adam launch.
"""

from __future__ import annotations

import numpy as np


def shard_by_rows(row_offsets, world: int) -> list[tuple[int, int]]:
    """Contiguous program ranges with ~equal step rows per rank."""
    off = np.asarray(row_offsets, dtype=np.int64)
    n = off.shape[0] - 1
    total = off[-1] - off[0]
    cuts = [0]
    for r in range(1, world):
        target = off[0] + total * r / world
        cuts.append(int(np.searchsorted(off, target, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def lpt_assign(task_sizes, world: int) -> list[list[int]]:
    """Longest-processing-time greedy on n_t^2; ties by task index (deterministic)."""
    sizes = np.asarray(task_sizes, dtype=np.int64)
    cost = sizes.astype(np.float64) ** 2
    order = sorted(range(len(sizes)), key=lambda t: (-cost[t], t))
    load = [0.0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for t in order:
        r = min(range(world), key=lambda q: (load[q], q))
        out[r].append(t)
        load[r] += cost[t]
    return [sorted(x) for x in out]


def dp_microbatch(perm, step: int, batch: int, rank: int, world: int) -> np.ndarray:
    """The rank's slice of global minibatch `step` (may be empty at the tail)."""
    lo = step * world * batch + rank * batch
    return np.asarray(perm[lo: lo + batch])


def dp_steps(n: int, batch: int, world: int) -> int:
    return (n + world * batch - 1) // (world * batch)


def global_max_int(x: int, group=None) -> int:
    """MAX of one integer over the ranks of `group`."""
    import torch
    import torch.distributed as dist

    v = torch.tensor([int(x)], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        v = v.cuda()
    dist.all_reduce(v, op=dist.ReduceOp.MAX, group=group)
    return int(v.item())


def mean_microbatch_gradient(grad, n_local: int, group=None):
    """All-reduce (sum) the local gradient and the count of non-empty
    microbatches; returns the mean over non-empty microbatches (in place).
    ``grad`` is a torch tensor; an empty microbatch must contribute zeros."""
    import torch
    import torch.distributed as dist

    cnt = torch.tensor([1.0 if n_local > 0 else 0.0], dtype=grad.dtype, device=grad.device)
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    grad /= cnt
    return grad


class DataParallelTunerEpoch:
    """One data-parallel training epoch of a RecurrentAttentionTuner replica.

    Per global step k: the rank's microbatch (dp_microbatch) runs the fused
    kernel in gradient mode (forward, rank/MSE loss, backward, fixed-order
    per-sample reduction), the flat fp32 gradient (330 KB for the default
    tuner) is all-reduced over NCCL, and the standalone fused Adam kernel
    applies the identical update on every replica.
    """

    def __init__(self, est, prog, y_dev, batch: int, group=None):
        import torch
        import torch.distributed as dist

        from . import _device

        self.est, self.prog, self.y, self.B, self.group = est, prog, y_dev, batch, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.dims = est._dims()
        self.flat = est._dev_params(self.dims).clone()
        self.m = torch.zeros_like(self.flat)
        self.v = torch.zeros_like(self.flat)
        self.t = 0
        self._dev = _device

    def run(self, perm: np.ndarray, lr: float, local_shard: bool = False) -> int:
        """Train over `perm`; returns the number of global steps taken.

        local_shard=False: `perm` is the global permutation (identical on every
        rank) and rank r takes slice r of each global minibatch.
        local_shard=True: every rank holds its own data shard and `perm` is a
        permutation of it; global step k uses each rank's k-th local slice."""
        import torch

        from . import _lib
        from .estimators import _BETA1, _BETA2, _EPS

        n = len(perm)
        perm_dev = self._dev.to_dev(np.asarray(perm, dtype=np.int32))
        if local_shard:
            # shards may differ in size: every rank loops to the LONGEST
            # shard's step count (ranks past their shard contribute zero
            # gradients and a zero count), so all ranks issue the same
            # collectives
            steps = global_max_int((n + self.B - 1) // self.B, self.group)
        else:
            steps = dp_steps(n, self.B, self.world)
        stream = self._dev.stream_ptr()
        for k in range(steps):
            lo = k * self.B if local_shard else k * self.world * self.B + self.rank * self.B
            cnt = max(0, min(self.B, n - lo))
            if cnt > 0:
                order = perm_dev[lo: lo + cnt]
                _, _, grad = self.est._launch_train(self.dims, self.flat, None, None, self.prog,
                                                    self.y, order, cnt, _lib.TT_MODE_GRAD, 0.0,
                                                    None, None)
            else:
                grad = torch.zeros_like(self.flat)
            mean_microbatch_gradient(grad, cnt, self.group)
            self.t += 1
            c1 = 1.0 - _BETA1**self.t
            c2 = 1.0 - _BETA2**self.t
            _lib.call("tt_adam_step_f32" if self.flat.dtype == torch.float32 else "tt_adam_step_f64",
                      self.flat.data_ptr(), grad.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                      self.flat.numel(), None, lr, _BETA1, _BETA2, _EPS, c1, c2, stream)
        return steps


def gather_counts(local_counts: dict, n_tasks: int, group=None) -> np.ndarray:
    """Combine per-task int64 counts computed on disjoint task sets."""
    import torch
    import torch.distributed as dist

    buf = torch.zeros(n_tasks, dtype=torch.int64)
    for t, c in local_counts.items():
        buf[t] = int(c)
    if dist.get_backend(group) == "nccl":
        buf = buf.cuda()
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf.cpu().numpy()


def exchange_handles(handle: bytes, group=None) -> list:
    """All-gather one 64-byte CUDA IPC handle per rank (rank order)."""
    import torch.distributed as dist

    if len(handle) != 64:
        raise ValueError("CUDA IPC handles are 64 bytes")
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, bytes(handle), group=group)
    return handles


class FusedDataParallelTuner:
    """One rank of the fused data-parallel epoch (tt_tuner_train_dp_f32).

    Every rank holds an equal-size shard; global step k uses each rank's k-th
    local microbatch (SURVEY §8e option A).  Inside the one training launch
    per epoch, each gradient job of the latency-path kernel stores its
    reduced parameter slice into the peers' exchange buffers (opened by CUDA
    IPC: NVLink peer memory on the box), raises a release flag there, waits
    for the peers' flags and sums the slots in rank order -- the update is
    bit-identical on every rank.  ``create`` wires the buffers over
    torch.distributed; ``local_group`` builds W ranks inside one process on
    one GPU (tests: the ranks run concurrently on disjoint SMs).
    """

    def __init__(self, est, prog, y_dev, batch: int, world: int, rank: int, xb, owned, group=None):
        import torch

        from . import _device

        self.est, self.prog, self.y, self.B = est, prog, y_dev, batch
        self.world, self.rank = world, rank
        self.group = group  # torch.distributed group (create) or None (local_group)
        self.dims = est._dims()
        self.flat = est._dev_params(self.dims).clone()
        self.m = torch.zeros_like(self.flat)
        self.v = torch.zeros_like(self.flat)
        self.xb = xb          # device int64 tensor [world] of buffer addresses
        self._owned = owned   # (pointer, is_ipc_mapping) to release
        self.gstep = 0
        self._dev = _device

    @staticmethod
    def _buffer_bytes(dims, world: int) -> int:
        from . import _lib

        n = _lib.load().tt_tuner_dp_buffer_bytes(dims["L"], dims["H"], dims["d0"], dims["C"], world)
        if n == 0:
            raise _lib.LibraryError("fused data parallel training needs hidden 32")
        return int(n)

    @staticmethod
    def _alloc(nbytes: int):
        import ctypes

        from . import _lib

        ptr = ctypes.c_void_p()
        handle = (ctypes.c_uint8 * 64)()
        _lib.call("tt_ipc_alloc", nbytes, ctypes.byref(ptr), handle)
        return int(ptr.value), bytes(handle)

    @classmethod
    def create(cls, est, prog, y_dev, batch: int, group=None):
        """Collective over torch.distributed: allocate this rank's exchange
        buffer, all-gather the IPC handles, open the peers' buffers.  Every
        rank takes part in every collective even when a step fails, and the
        ranks agree on the outcome (LibraryError on all of them if any
        failed: e.g. no peer access between the GPUs)."""
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _device, _lib

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        ok, own, handle, owned = True, None, bytes(64), []
        try:
            own, handle = cls._alloc(cls._buffer_bytes(est._dims(), world))
            owned.append((own, False))
        except Exception:  # noqa: BLE001
            ok = False
        handles = exchange_handles(handle, group)
        ptrs = []
        if ok:
            try:
                for r, h in enumerate(handles):
                    if r == rank:
                        ptrs.append(own)
                        continue
                    p = ctypes.c_void_p()
                    _lib.call("tt_ipc_open", (ctypes.c_uint8 * 64).from_buffer_copy(h), ctypes.byref(p))
                    ptrs.append(int(p.value))
                    owned.append((int(p.value), True))
            except Exception:  # noqa: BLE001
                ok = False
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                            device=_device.device() if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()) == 0:
            for ptr, mapped in owned:
                try:
                    _lib.call("tt_ipc_close" if mapped else "tt_dev_free", ptr)
                except Exception:  # noqa: BLE001
                    pass
            raise _lib.LibraryError("fused data parallel: peer exchange buffers unavailable on some rank")
        xb = torch.tensor(ptrs, dtype=torch.int64, device=_device.device())
        return cls(est, prog, y_dev, batch, world, rank, xb, owned, group=group)

    @classmethod
    def local_group(cls, ests, progs, ys, batch: int):
        """W ranks in this process on one GPU (plain device buffers)."""
        import torch

        from . import _device

        world = len(ests)
        nbytes = cls._buffer_bytes(ests[0]._dims(), world)
        bufs = [cls._alloc(nbytes)[0] for _ in range(world)]
        xb = torch.tensor(bufs, dtype=torch.int64, device=_device.device())
        return [cls(e, p, y, batch, world, r, xb, [(bufs[r], False)])
                for r, (e, p, y) in enumerate(zip(ests, progs, ys))]

    def preconditions(self, n: int) -> tuple[int, int, int]:
        """(steps of this launch, global step base, latency-path eligible):
        every rank's kernel waits on its peers' slices for every step, so
        these must agree across ranks before anything is launched."""
        from . import _lib

        d = self.dims
        ok = _lib.load().tt_tuner_train_fast_eligible(d["L"], d["H"], d["heads"], d["U"], d["d0"],
                                                       d["C"], self.prog.max_steps, self.B)
        return (n + self.B - 1) // self.B, self.gstep, int(ok)

    def _agree(self, pre: tuple[int, int, int]) -> None:
        """All-reduce the preconditions (MIN and MAX in one MAX collective)
        and raise LibraryError on EVERY rank if any rank differs or is not
        eligible, so no rank launches a kernel its peers would wait on."""
        import torch
        import torch.distributed as dist

        from . import _lib

        if self.group is None or not dist.is_initialized():
            return
        v = torch.tensor(list(pre) + [-x for x in pre], dtype=torch.int64)
        if dist.get_backend(self.group) == "nccl":
            v = v.to(self._dev.device())
        dist.all_reduce(v, op=dist.ReduceOp.MAX, group=self.group)
        v = v.cpu().tolist()
        hi, lo = v[:3], [-x for x in v[3:]]
        if hi != lo or lo[2] != 1:
            raise _lib.LibraryError(
                f"fused data parallel: ranks disagree or are not eligible "
                f"(steps {lo[0]}..{hi[0]}, step base {lo[1]}..{hi[1]}, eligible min {lo[2]}); "
                "every rank needs an equal-size shard, the same step count so far and programs "
                "the latency-path kernel accepts")

    def run(self, perm: np.ndarray, lr: float):
        """Enqueue one epoch over this rank's shard in the order `perm` (equal
        length on every rank) on the current stream; returns the device
        status [first non-finite step or -1, abort word] (check_status)."""
        from . import _lib
        from .estimators import _BETA1, _BETA2, _EPS, _bias_corrections

        d, est, prog = self.dims, self.est, self.prog
        n = len(perm)
        pre = self.preconditions(n)
        self._agree(pre)
        if pre[2] != 1:
            raise _lib.LibraryError("fused data parallel: not eligible for the latency-path kernel")
        n_steps = pre[0]
        lib = _lib.load()
        nbytes = lib.tt_tuner_train_workspace_bytes(0, d["L"], d["H"], d["d0"], d["C"], prog.max_steps,
                                                    self.B)
        ws = self._dev.workspace(nbytes, "tuner_train_dp")
        order = self._dev.to_dev(np.asarray(perm, dtype=np.int32))
        corr = self._dev.to_dev(_bias_corrections(self.gstep, n_steps))
        self.step_loss = self._dev.empty(n_steps, self.flat.dtype)
        status = self._dev.to_dev(np.array([-1, 0], dtype=np.int32))
        loss_kind = _lib.TT_LOSS_RANK if est.loss == "ranking" else _lib.TT_LOSS_MSE
        _lib.call("tt_tuner_train_dp_f32", self.flat.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                  prog.steps.data_ptr(), prog.offsets.data_ptr(), prog.ctx.data_ptr(), self.y.data_ptr(),
                  order.data_ptr(), n, self.B, loss_kind, float(lr), _BETA1, _BETA2, _EPS,
                  corr.data_ptr(), None, d["L"], d["H"], d["heads"], d["U"], d["d0"], d["C"],
                  prog.max_steps, self.world, self.rank, self.gstep, self.xb.data_ptr(),
                  self.step_loss.data_ptr(), status.data_ptr(), ws.data_ptr(), nbytes,
                  self._dev.stream_ptr())
        self.gstep += n_steps
        self._keep = (order, corr)  # alive until the launch completes
        return status

    @staticmethod
    def check_status(status) -> int:
        """Raise if the launch's exchange timed out waiting for a peer;
        return the first non-finite step (-1 if none)."""
        from . import _lib

        s = status.cpu().tolist()
        if len(s) > 1 and s[1] != 0:
            raise _lib.LibraryError("fused data parallel: a peer did not deliver its gradient slice "
                                    "within the timeout (dead or diverged rank); parameters are invalid")
        return int(s[0])

    def close(self):
        from . import _lib

        for ptr, mapped in self._owned:
            _lib.call("tt_ipc_close" if mapped else "tt_dev_free", ptr)
        self._owned = []


# ------------------------------------------------ sharded scoring / PCA --


def _group_info(group):
    import torch.distributed as dist

    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _all_gather_host(obj, group):
    import torch.distributed as dist

    world, _ = _group_info(group)
    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj, group=group)
    return out


def sharded_predict(est, sequences, group=None, gather: bool = True, predict_fn=None):
    """Config-3 search-time/bulk scoring sharded by program:
    every rank passes the same candidate list; rank r packs and scores only
    its contiguous range of ~equal step rows (shard_by_rows on the step
    counts) with the estimator's own kernels -- no collective on the data
    path.  gather=True reassembles the float64 scores on every rank with one
    host all-gather of the slices (the reference's ``predict`` result,
    tuner.py:468-476); gather=False returns (lo, hi, local_scores).

    ``predict_fn(est, seqs) -> np.ndarray`` defaults to ``est.predict``
    (tests inject the oracle to exercise the sharding on CPU)."""
    world, rank = _group_info(group)
    n = len(sequences)
    lens = np.fromiter((len(s.steps) for s in sequences), dtype=np.int64, count=n)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    lo, hi = shard_by_rows(off, world)[rank]
    fn = predict_fn or (lambda e, s: e.predict(s))
    local = np.asarray(fn(est, sequences[lo:hi]), dtype=np.float64) if hi > lo else np.zeros(0)
    if not gather:
        return lo, hi, local
    parts = _all_gather_host((lo, hi, local), group)
    out = np.empty(n, dtype=np.float64)
    for a, b, v in parts:
        out[a:b] = v
    return out


def sharded_pca_counts(y, y_hat, task_offsets, group=None, count_fn=None) -> np.ndarray:
    """Config-4 PCA sharded by task: tasks are assigned to ranks
    by LPT on n_t^2 (lpt_assign), every rank counts its tasks' concordant
    pairs with K1 (one launch over its tasks), and ONE all-reduce of the
    zero-initialised per-task int64 vector combines them (gather_counts).
    Counts are exact integers, so the result is identical to the unsharded
    count whatever the assignment.  Every rank passes the full (y, y_hat,
    task_offsets); returns the per-task counts on every rank.

    ``count_fn(y, y_hat, offsets) -> int64 counts`` defaults to the GPU
    pca_counts (tests inject the oracle)."""
    from .metrics import pca_counts

    world, rank = _group_info(group)
    off = np.asarray(task_offsets, dtype=np.int64)
    sizes = np.diff(off)
    n_tasks = sizes.shape[0]
    mine = [t for t in lpt_assign(sizes, world)[rank] if sizes[t] >= 2]
    local: dict = {}
    if mine:
        idx = np.concatenate([np.arange(off[t], off[t + 1]) for t in mine])
        sub = np.zeros(len(mine) + 1, dtype=np.int64)
        np.cumsum(sizes[mine], out=sub[1:])
        yy = np.asarray(y, dtype=np.float64)[idx]
        ss = np.asarray(y_hat, dtype=np.float64)[idx]
        c = (count_fn or pca_counts)(yy, ss, sub)
        local = {t: int(v) for t, v in zip(mine, c)}
    if world == 1:
        out = np.zeros(n_tasks, dtype=np.int64)
        for t, v in local.items():
            out[t] = v
        return out
    return gather_counts(local, n_tasks, group)


def sharded_segmented_pca(y, y_hat, task_offsets, group=None, count_fn=None) -> np.ndarray:
    """Per-task PCA values (NaN for tasks with < 2 records) from the sharded
    counts; float(correct)/float(total) equals the reference's mean bit for bit."""
    from .metrics import pca_from_counts

    return pca_from_counts(sharded_pca_counts(y, y_hat, task_offsets, group, count_fn), task_offsets)
