"""Data-parallel plumbing for batch-sharded convolution training steps
(north_star: the batch dimension is split over the GPUs of one node and the
weight gradients are all-reduced with NCCL; BASELINE.json configs[4]).

* ``shard_batch`` — the contiguous image range of one rank.
* ``DataParallel`` — the product path: a ctypes mirror of the native
  ``primkit_dp_*`` C ABI (csrc/host/dp.cpp). Gradients are registered in
  backward order, grouped into fp32 buckets and all-reduced by NCCL on a comm
  stream as soon as each bucket's last backward-weights kernel is enqueued,
  overlapping the rest of the backward pass. torch.distributed is only used
  to broadcast the 128-byte NCCL unique id.
* ``GradBucket`` — a host-side restatement of the same bucket semantics
  (fp32 sum of per-rank gradients) over any torch.distributed backend; the
  CPU (gloo) tests use it to pin what the native path computes.
"""
from __future__ import annotations

import ctypes as C


def shard_batch(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """(first image, image count) of `rank`'s contiguous shard; remainders go
    to the lowest ranks so shard sizes differ by at most one image."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(global_batch, world)
    count = base + (1 if rank < rem else 0)
    start = rank * base + min(rank, rem)
    return start, count


class DataParallel:
    """Native NCCL gradient buckets (primkit_dp_*) bound to a primkit handle."""

    def __init__(self, lib, handle_ptr, rank: int, world: int, dist=None, average=False,
                 bucket_bytes: int | None = None):
        self.L = lib
        uid = C.create_string_buffer(128)
        if rank == 0:
            lib.check(lib.lib.primkit_dp_unique_id(uid))
        if dist is not None and world > 1:
            box = [bytes(uid.raw)]
            dist.broadcast_object_list(box, src=0)
            uid = C.create_string_buffer(box[0], 128)
        self.ptr = C.c_void_p()
        lib.check(lib.lib.primkit_dp_create(handle_ptr, uid, world, rank, int(average),
                                            C.byref(self.ptr)))
        if bucket_bytes:
            lib.check(lib.lib.primkit_dp_set_bucket_bytes(self.ptr, bucket_bytes))

    def register(self, tensor, etype) -> int:
        idx = C.c_int()
        self.L.check(self.L.lib.primkit_dp_register(self.ptr, C.c_void_p(tensor.data_ptr()),
                                                    tensor.numel(), etype, C.byref(idx)))
        return idx.value

    def ready(self, index: int):
        self.L.check(self.L.lib.primkit_dp_grad_ready(self.ptr, index))

    def finish(self):
        self.L.check(self.L.lib.primkit_dp_finish(self.ptr))

    def check(self):
        self.L.check(self.L.lib.primkit_dp_check(self.ptr))

    def buckets(self) -> int:
        n = C.c_int()
        self.L.check(self.L.lib.primkit_dp_buckets(self.ptr, C.byref(n)))
        return n.value

    def bucket_of(self, index: int) -> int:
        b = C.c_int()
        self.L.check(self.L.lib.primkit_dp_bucket_of(self.ptr, index, C.byref(b)))
        return b.value

    def close(self):
        if self.ptr:
            self.L.lib.primkit_dp_destroy(self.ptr)
            self.ptr = C.c_void_p()


class GradBucket:
    """Packs per-layer gradients into one flat fp32 buffer, all-reduces it
    (sum) and writes the result back in each tensor's dtype — the semantics
    of one native bucket, for any torch.distributed backend."""

    def __init__(self, torch, tensors):
        self.torch = torch
        self.tensors = list(tensors)
        total = sum(t.numel() for t in self.tensors)
        self.flat = torch.empty(total, dtype=torch.float32, device=self.tensors[0].device)

    def pack(self):
        off = 0
        for t in self.tensors:
            n = t.numel()
            self.flat[off:off + n].copy_(t.reshape(-1))
            off += n

    def unpack(self):
        off = 0
        for t in self.tensors:
            n = t.numel()
            t.copy_(self.flat[off:off + n].view(t.shape))
            off += n

    def allreduce(self, dist, group=None):
        self.pack()
        dist.all_reduce(self.flat, group=group)
        self.unpack()
