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


class ShardPlan:
    """This rank's part of a globally batched layer step (bench.py, chain.py).

    * ``start``/``count``: the contiguous image range (``shard_range``);
    * ``shape(g)``: the local ``conv_shape`` (batch = count) of a global one;
    * ``slice_nchwc(t)``: the rank's images of a GLOBAL ActNCHWc tensor as a
      view -- ActNCHWc keeps the batch outermost (P/include/spconv/tensor.hpp
      act_index), so a shard is one contiguous element range, no copy;
    * ``global_flops(shapes)``: dense-equivalent FLOPs of the whole job.

    ActCHWNn is NOT sliced (its 16-image lane blocks interleave the batch);
    each rank packs its own shard, and a shard of n < 16 images leaves zero
    lanes the zero check skips (P/src/tensor.cpp:94-108)."""

    def __init__(self, n_global: int, world: int = 1, rank: int = 0):
        self.n_global, self.world, self.rank = n_global, world, rank
        self.start, self.count = shard_range(n_global, world, rank)

    def shape(self, global_shape):
        return global_shape.with_batch(self.count)

    def slice_nchwc(self, t):
        from .api import BlockedTensor, Layout, SpconvError
        if t.layout != Layout.act_nchwc or t.n != self.n_global:
            raise SpconvError(3, "slice_nchwc: need the global ActNCHWc tensor")
        per = t.c * t.h * t.w
        data = t.data.reshape(-1)[self.start * per:(self.start + self.count) * per]
        return BlockedTensor(Layout.act_nchwc, t.V, self.count, t.c, t.h, t.w, data=data)

    def slice_plain(self, x):
        return x[self.start:self.start + self.count]

    def global_flops(self, shapes) -> int:
        return sum(sh.with_batch(self.n_global).dense_flops() for sh in shapes)


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


class DeviceBuffer:
    """A raw device allocation (e.g. an NCCL symmetric window) presented with
    the two methods the pass wrappers use: ``data_ptr()`` and ``numel()``."""

    def __init__(self, ptr: int, numel: int, owner=None):
        self._ptr, self._numel, self._owner = int(ptr), int(numel), owner

    def data_ptr(self) -> int:
        return self._ptr

    def numel(self) -> int:
        return self._numel

    def slice(self, start: int, count: int) -> "DeviceBuffer":
        return DeviceBuffer(self._ptr + 4 * start, count, self._owner)


class Comm:
    """The product's NCCL communicator (``spc_comm``, csrc/comm.cu) for the
    BWW weight-gradient exchange, one rank per GPU on the current device.

    Rank 0 draws the NCCL unique id through the C ABI; it reaches the other
    ranks over the existing torch.distributed group (any backend), then
    every rank calls ``spc_comm_init``.  ``allreduce`` enqueues the in-place
    fp32 sum (``spc_bww_allreduce``) on a stream with no host sync;
    ``window`` allocates dG storage as an NCCL symmetric window."""

    def __init__(self, group=None):
        import ctypes as C

        import torch.distributed as dist

        from . import _lib
        self._C = C
        self.L = _lib.load()
        self.rank, self.size = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_ubyte * 128)()
        if self.rank == 0:
            self._check(self.L.spc_comm_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        self._check(self.L.spc_comm_init(C.byref(h), self.size, uid, self.rank))
        self.h = h
        self.nccl = self.L.spc_comm_nccl(h)
        self._windows = []

    def _check(self, st):
        from . import _lib
        from .api import SpconvError
        if st:
            raise SpconvError(st, _lib.last_error())

    def window(self, numel: int):
        """Collective: a float32 device buffer in an NCCL symmetric window
        (``(DeviceBuffer, True)``); where NCCL cannot provide one, plain NCCL
        memory (``(DeviceBuffer, False)``) or, if even that fails, a torch
        CUDA tensor (``(tensor, False)``) -- the allreduce works on all three."""
        C = self._C
        p, sym = C.c_void_p(), C.c_int()
        if self.L.spc_comm_window_alloc(self.h, 4 * numel, C.byref(p), C.byref(sym)) != 0:
            import torch
            return torch.zeros(numel, dtype=torch.float32, device="cuda"), False
        buf = DeviceBuffer(p.value, numel, self)
        self._windows.append(p)
        return buf, bool(sym.value)

    def allreduce(self, buf, stream_ptr: int, start: int = 0, count: int | None = None) -> None:
        """In-place fp32 sum of buf[start:start+count] across the ranks, on `stream_ptr`."""
        C = self._C
        n = buf.numel() - start if count is None else count
        self._check(self.L.spc_bww_allreduce(C.c_void_p(self.nccl), C.c_void_p(buf.data_ptr() + 4 * start), n,
                                             C.c_void_p(stream_ptr)))

    def close(self) -> None:
        if getattr(self, "h", None) is not None:
            self._check(self.L.spc_comm_destroy(self.h))
            self.h = None


class CommAllreduce:
    """GradAllreduce's interface (submit / wait) over the product's
    communicator: each submitted dG slice is summed in place by
    ``spc_bww_allreduce`` on a side stream that waits for the producer, so
    the exchange of block b overlaps the backward of block b-1."""

    def __init__(self, comm: Comm, device=None):
        import torch
        self.comm = comm
        self.stream = torch.cuda.Stream(device=device)

    def submit(self, grad, producer_stream=None):
        import torch
        if self.comm.size == 1:
            return
        ev = torch.cuda.Event()
        ev.record(producer_stream or torch.cuda.current_stream())
        self.stream.wait_event(ev)
        self.comm.allreduce(grad, self.stream.cuda_stream)

    def wait(self, consumer_stream=None):
        import torch
        (consumer_stream or torch.cuda.current_stream()).wait_stream(self.stream)
