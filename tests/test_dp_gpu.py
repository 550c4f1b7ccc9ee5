"""Data-parallel dW all-reduce (north_star) on one B200.

* The native NCCL bucket layer (primkit_dp_*, csrc/host/dp.cpp) with a
  1-rank communicator: bucket grouping in backward order, pack -> ncclAllReduce
  -> unpack on the comm stream, the join in finish(), and the whole sequence
  captured into a CUDA graph together with the product's wgrad kernels. A
  1-rank sum is the identity, so dW must come back bit-identical (bf16 -> fp32
  -> bf16 is exact).
* The sharding semantics with the product kernels: two processes on the same
  GPU each run the product backward-weights kernel on their half of the batch;
  the fp32 sum of the two shards (gloo over host copies, since NCCL refuses two
  ranks on one device) matches the oracle's full-batch conv_backward_weights
  (proj/src/core/conv.cpp:801-873) within the bf16 tolerance.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

LAYERS = [dict(c=64, k=64, h=56, r=3, pad=1, stride=1), dict(c=256, k=512, h=28, r=1, pad=0, stride=1),
          dict(c=128, k=128, h=56, r=3, pad=1, stride=2), dict(c=512, k=2048, h=7, r=1, pad=0, stride=1)]


def _stream_handle(lib):
    h = C.c_void_p()
    lib.check(lib.lib.primkit_handle_create_with_stream(
        C.c_void_p(torch.cuda.current_stream().cuda_stream), 0, C.byref(h)))
    return h


def _wgrad_problem(L, n):
    return problem(n=n, c=L["c"], h=L["h"], w=L["h"], k=L["k"], y=L["r"], x=L["r"], pad=L["pad"],
                   stride=L["stride"], direction=abi.BACKWARD_WEIGHTS, etype=abi.BF16)


def _run(lib, h, p, a, b, out):
    ws = C.c_uint64()
    lib.check(lib.lib.primkit_conv_device_workspace(h, C.byref(p), b"Im2colGemm", C.byref(ws)))
    wsb = torch.empty(max(int(ws.value), 256), dtype=torch.uint8, device="cuda")
    lib.check(lib.lib.primkit_conv_run_device(h, C.byref(p), b"Im2colGemm", C.c_void_p(a.data_ptr()),
                                              C.c_void_p(b.data_ptr()), C.c_void_p(out.data_ptr()),
                                              C.c_void_p(wsb.data_ptr()), C.c_size_t(wsb.numel())))
    return wsb


def test_native_buckets_single_rank_graph(lib):
    from paper_1910_00078_b200.dist import DataParallel
    h = _stream_handle(lib)
    n = 32
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    rnd = lambda s: (torch.rand(s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa: E731
    ops, grads = [], []
    for L in LAYERS:
        ho = (L["h"] + 2 * L["pad"] - L["r"]) // L["stride"] + 1
        dy, x = rnd((n, ho, ho, L["k"])), rnd((n, L["h"], L["h"], L["c"]))
        dw = torch.zeros((L["k"], L["r"], L["r"], L["c"]), dtype=torch.bfloat16, device="cuda")
        ops.append((_wgrad_problem(L, n), dy, x, dw))
        grads.append(dw)
    dp = DataParallel(lib, h, rank=0, world=1, bucket_bytes=4 << 20)  # several buckets
    for dw in grads:
        dp.register(dw, abi.BF16)
    sizes = [dw.numel() * 4 for dw in grads]
    owners = [dp.bucket_of(i) for i in range(len(grads))]
    assert owners == sorted(owners) and owners[0] == 0 and dp.buckets() == owners[-1] + 1
    assert dp.buckets() >= 2, (sizes, owners)

    def step():
        keep = []
        for i, (p, dy, x, dw) in enumerate(ops):
            keep.append(_run(lib, h, p, dy, x, dw))
            dp.ready(i)
        dp.finish()
        return keep

    keep = step()  # eager
    torch.cuda.synchronize()
    dp.check()
    eager = [dw.clone() for dw in grads]
    for dw in grads:
        dw.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        lib.check(lib.lib.primkit_handle_set_stream(h, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        keep = step()
    lib.check(lib.lib.primkit_handle_set_stream(h, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    graph.replay()
    torch.cuda.synchronize()
    dp.check()
    for a, b in zip(eager, grads):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))  # 1-rank sum = identity, deterministic
    # and the values are the backward-weights result (oracle, sampled)
    p, dy, x, dw = ops[0]
    hst = lambda t: t.view(torch.int16).cpu().numpy().view(np.uint16)  # noqa: E731
    rng = np.random.default_rng(1)
    ks, taps = rng.choice(64, 16, replace=False), np.stack([rng.integers(0, 3, 32), rng.integers(0, 3, 32),
                                                             rng.integers(0, 64, 32)], 1)
    want = oracle.sample_backward_weights(p, hst(dy), hst(x), ks, taps).ravel()
    got = hst(dw)[ks[:, None], taps[None, :, 0], taps[None, :, 1], taps[None, :, 2]]
    got = (got.astype(np.uint32) << 16).view(np.float32).ravel()
    assert rel_l2(got, want) <= 1e-2
    del keep
    dp.close()
    lib.lib.primkit_handle_destroy(h)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_worker(rank, world, port, q):
    import torch as T
    import torch.distributed as dist

    from paper_1910_00078_b200.dist import GradBucket, shard_batch
    from paper_1910_00078_b200.primkit import library
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = library()
    T.cuda.set_device(0)
    h = _stream_handle(lib)
    rng = np.random.default_rng(17)
    n = 16
    results = []
    for L in LAYERS[:3]:
        ho = (L["h"] + 2 * L["pad"] - L["r"]) // L["stride"] + 1
        dy = oracle.round_bf16(rng.uniform(-1, 1, (n, ho, ho, L["k"])).astype(np.float32))
        x = oracle.round_bf16(rng.uniform(-1, 1, (n, L["h"], L["h"], L["c"])).astype(np.float32))
        s0, cnt = shard_batch(n, rank, world)
        dyd = T.from_numpy(dy[s0:s0 + cnt].copy()).cuda().to(T.bfloat16)
        xd = T.from_numpy(x[s0:s0 + cnt].copy()).cuda().to(T.bfloat16)
        dw = T.empty((L["k"], L["r"], L["r"], L["c"]), dtype=T.bfloat16, device="cuda")
        _run(lib, h, _wgrad_problem(L, cnt), dyd, xd, dw)
        T.cuda.synchronize()
        g = dw.cpu()  # product kernel's per-shard dW
        GradBucket(T, [g]).allreduce(dist)  # fp32 sum over the shards
        results.append((L, dy, x, g.float().numpy()))
    if rank == 0:
        errs = []
        for L, dy, x, got in results:
            p = problem(n=n, c=L["c"], h=L["h"], w=L["h"], k=L["k"], y=L["r"], x=L["r"], pad=L["pad"],
                        stride=L["stride"])
            full = oracle.conv_backward_weights(p, dy.transpose(0, 3, 1, 2), x.transpose(0, 3, 1, 2))
            errs.append(rel_l2(got.transpose(0, 3, 1, 2), full))
        q.put(max(errs))
    lib.lib.primkit_handle_destroy(h)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_product_wgrad_sum_matches_full_batch_oracle():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) <= 1e-2
