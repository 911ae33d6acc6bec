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
  formed by one all-reduce before the (replicated) fused Adam update.
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
