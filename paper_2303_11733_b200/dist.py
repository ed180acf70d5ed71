"""Multi-GPU plumbing for the DIPPM path (one process per GPU, torch.distributed).

Graphs are independent, so:
  * inference shards contiguous graph ranges across ranks, balanced by node
    count (the forward's cost is linear in N), with no collective
    on the hot path; `gather_predictions` optionally collects (y, mig) on every
    rank (16 B/graph);
  * training is data parallel: each rank computes its batch's gradient share
    on device, ONE all-reduce (sum) of the flat fp32 gradient vector is the
    only exchange, and the Huber kernel's gradient denominator is the GLOBAL
    batch size so the sum over ranks is exactly the global batch mean of
    gnn.backward (gnn.py:402-404) even when per-rank batches differ.
Backend: "nccl" on GPUs (NVLink/NVSwitch); "gloo" in the CPU tests.
"""

from __future__ import annotations

import numpy as np


def shard_by_nodes(node_counts, world: int) -> list:
    """Contiguous graph ranges [(start, end)] per rank with ~equal total nodes.

    Cut points are the graph boundaries closest to the cumulative-node quantiles
    k/world; every graph is assigned exactly once and order is preserved."""
    n = np.asarray(node_counts, dtype=np.int64)
    if world < 1:
        raise ValueError("world size must be >= 1")
    cum = np.concatenate([[0], np.cumsum(n)])
    total = cum[-1]
    cuts = [0]
    for k in range(1, world):
        target = total * k / world
        i = int(np.searchsorted(cum, target))
        if i > 0 and (i >= len(cum) or abs(cum[i - 1] - target) <= abs(cum[i] - target)):
            i -= 1
        cuts.append(min(max(i, cuts[-1]), len(n)))
    cuts.append(len(n))
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def global_batch_size(local: int, group=None) -> int:
    """Sum of per-rank batch sizes (one tiny all-reduce; the training denominator)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([local], dtype=torch.int64, device=dev)
    dist.all_reduce(t, group=group)
    return int(t.item())


def allreduce_sum(tensor, group=None):
    """In-place sum over ranks (the DP gradient exchange)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, group=group)
    return tensor


class OverlappedAllReduce:
    """The DP gradient exchange split in two buckets so the first overlaps the backward.

    The flat gradient layout is sage1 | sage2 | sage3 | fc1..fc3 (gnn.py:488-491), and the
    backward finishes fc* and sage3 first: `begin(grads[off:])` is issued right after the
    layer-3 weight gradient (NCCL orders it after the work already queued on the compute
    stream and runs it on its own stream while the layer-2/1 backward proceeds), the
    remaining bucket follows the backward, and `finish()` makes the compute stream wait for
    both before Adam.  Calling the object on a tensor is a plain blocking all-reduce."""

    def __init__(self, group=None):
        self.group = group
        self.works = []

    def _active(self):
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1

    def begin(self, tensor) -> None:
        import torch.distributed as dist
        if self._active():
            self.works.append(dist.all_reduce(tensor, group=self.group, async_op=True))

    def finish(self) -> None:
        for w in self.works:
            w.wait()
        self.works.clear()

    def __call__(self, tensor):
        self.begin(tensor)
        self.finish()
        return tensor


def gather_predictions(y, mig, group=None):
    """All-gather variable-length per-rank (y [g,3], mig [g]) arrays in rank order."""
    import torch
    import torch.distributed as dist
    y = torch.as_tensor(y)
    mig = torch.as_tensor(mig)
    if not (dist.is_available() and dist.is_initialized()):
        return y, mig
    world = dist.get_world_size(group)
    n = torch.tensor([y.shape[0]], dtype=torch.int64, device=y.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    m = int(max(s.item() for s in sizes))
    yp = torch.zeros(m, 3, dtype=y.dtype, device=y.device)
    yp[:y.shape[0]] = y
    mp = torch.full((m,), -1, dtype=torch.int32, device=y.device)
    mp[:mig.shape[0]] = mig.to(torch.int32)
    ys = [torch.zeros_like(yp) for _ in range(world)]
    ms = [torch.zeros_like(mp) for _ in range(world)]
    dist.all_gather(ys, yp, group=group)
    dist.all_gather(ms, mp, group=group)
    ys = torch.cat([t[:int(s.item())] for t, s in zip(ys, sizes)])
    ms = torch.cat([t[:int(s.item())] for t, s in zip(ms, sizes)]).to(torch.int8)
    return ys, ms
