"""Batch-sharded data parallelism on CPU (gloo, world size 2): shards cover
the batch exactly once, and the all-reduced per-shard dW equals the
full-batch backward-weights result (the oracle), which is what the NCCL path
in bench.py relies on."""
import os
import socket

import numpy as np
import pytest

from paper_1910_00078_b200.dist import shard_batch


def test_shard_batch_covers_batch():
    for n in (1, 7, 256, 1000):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, c = shard_batch(n, r, world)
                seen.extend(range(s, s + c))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard_batch(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1910_00078_b200.dist import GradBucket
    from paper_1910_00078_b200.primkit import problem

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(3)
    n = 5
    shapes = [dict(c=4, k=6, h=8, y=3, pad=1, stride=1), dict(c=6, k=4, h=8, y=1, pad=0, stride=2)]
    xs = [rng.uniform(-1, 1, (n, s["c"], s["h"], s["h"])).astype(np.float32) for s in shapes]
    dys = []
    for s in shapes:
        o = (s["h"] + 2 * s["pad"] - s["y"]) // s["stride"] + 1
        dys.append(rng.uniform(-1, 1, (n, s["k"], o, o)).astype(np.float32))
    start, cnt = shard_batch(n, rank, world)
    grads = []
    for s, x, dy in zip(shapes, xs, dys):
        p = problem(n=cnt, c=s["c"], h=s["h"], w=s["h"], k=s["k"], y=s["y"], x=s["y"],
                    pad=s["pad"], stride=s["stride"])
        grads.append(torch.from_numpy(oracle.conv_backward_weights(
            p, dy[start:start + cnt], x[start:start + cnt]).astype(np.float64)))
    bucket = GradBucket(torch, grads)
    bucket.allreduce(dist)
    if rank == 0:
        errs = []
        for s, x, dy, g in zip(shapes, xs, dys, grads):
            p = problem(n=n, c=s["c"], h=s["h"], w=s["h"], k=s["k"], y=s["y"], x=s["y"],
                        pad=s["pad"], stride=s["stride"])
            full = oracle.conv_backward_weights(p, dy, x).astype(np.float64)
            errs.append(float(np.max(np.abs(g.numpy() - full) / np.maximum(1, np.abs(full)))))
        q.put(max(errs))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_dw_allreduce_matches_full_batch():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) <= 1e-5


def test_bench_spawns_ranks_for_gpus_flag():
    """`bench.py --gpus 2` without a launcher re-runs itself under
    torch.distributed.run with 2 ranks (world size asserted == --gpus) and
    rank 0 prints the reduced line (gloo self-test, no GPU needed)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--launch-selftest"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]
    assert lines == [{"launch_selftest": True, "n_gpus": 2, "max_over_ranks": 2.0}]


def test_grad_bucket_reduces_in_fp32():
    """The bucket sums bf16 gradients in fp32 (one rounding at unpack), not in
    bf16 (error growing with world size)."""
    import torch
    from paper_1910_00078_b200.dist import GradBucket
    t = [torch.tensor([1.0, 256.0], dtype=torch.bfloat16), torch.tensor([3.0], dtype=torch.float32)]
    b = GradBucket(torch, t)
    assert b.flat.dtype == torch.float32

    class _Sum8:  # stands in for an 8-rank sum of identical shards
        @staticmethod
        def all_reduce(x, group=None):
            x.mul_(8)
    b.allreduce(_Sum8)
    assert t[0].tolist() == [8.0, 2048.0] and t[1].tolist() == [24.0]
