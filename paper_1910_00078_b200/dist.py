"""Data-parallel plumbing for batch-sharded convolution training steps
(north_star: the batch dimension is split over the GPUs of one node and the
weight gradients are all-reduced; BASELINE.json cfg5).

One process per GPU (torchrun), torch.distributed over NCCL on the B200 box;
the same code runs over gloo for the CPU tests. The only collective is the
all-reduce of the flat dW bucket."""
from __future__ import annotations


def shard_batch(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """(first image, image count) of `rank`'s contiguous shard; remainders go
    to the lowest ranks so shard sizes differ by at most one image."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(global_batch, world)
    count = base + (1 if rank < rem else 0)
    start = rank * base + min(rank, rem)
    return start, count


class GradBucket:
    """Packs per-layer dW tensors into one flat buffer so the step issues a
    single all-reduce (one NCCL launch; bucket sized for launch latency, not
    link count, on NVSwitch)."""

    def __init__(self, torch, tensors):
        self.torch = torch
        self.tensors = list(tensors)
        total = sum(t.numel() for t in self.tensors)
        dev = self.tensors[0].device
        self.flat = torch.empty(total, dtype=self.tensors[0].dtype, device=dev)

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
            t.copy_(self.flat[off:off + n].view_as(t))
            off += n

    def allreduce(self, dist, group=None):
        self.pack()
        dist.all_reduce(self.flat, group=group)
        self.unpack()
