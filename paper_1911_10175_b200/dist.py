"""Batch-sharded multi-GPU execution (one process per GPU, torch.distributed).

The reference has no distributed layer.  BASELINE.json
asks for work "partitioned over the batch dimension across 1/2/4/8 GPUs":

* FWD and BWI are independent per image: each rank runs its batch shard with
  no communication (ActNCHWc keeps the batch outermost, so a shard is one
  contiguous slice).
* BWW is a sum over images: each rank computes the partial dG of its shard
  and the ranks allreduce (sum, fp32) -- over NCCL/NVLink on GPUs.  That is
  the only exchange step of the path.

The ActCHWNn form of a shard is packed per rank (a shard of n < 16 images
leaves zero lanes, which the zero check skips for free).
"""
from __future__ import annotations


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous batch shard [start, start+count) of rank `rank`; sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def shard_batch(x, world: int, rank: int):
    """Rank's slice of a plain (n, c, h, w) array or tensor."""
    s, c = shard_range(x.shape[0], world, rank)
    return x[s:s + c]


class GradAllreduce:
    """Sum per-layer weight gradients across ranks, bucketed per layer and
    issued on a side stream so the exchange of layer l overlaps the passes
    that follow it.  On CPU (gloo) the side stream is unused."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.cuda = device is not None and torch.device(device).type == "cuda"
        self.stream = torch.cuda.Stream(device=device) if self.cuda else None
        self.pending = []

    def submit(self, grad, producer_stream=None):
        import torch
        if self.dist.get_world_size(self.group) == 1:
            return
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(producer_stream or torch.cuda.current_stream())
            self.stream.wait_event(ev)
            with torch.cuda.stream(self.stream):
                self.pending.append(self.dist.all_reduce(grad, group=self.group, async_op=True))
        else:
            self.pending.append(self.dist.all_reduce(grad, group=self.group, async_op=True))

    def wait(self, consumer_stream=None):
        import torch
        for w in self.pending:
            w.wait()
        self.pending.clear()
        if self.cuda:
            (consumer_stream or torch.cuda.current_stream()).wait_stream(self.stream)
