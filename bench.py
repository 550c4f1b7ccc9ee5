#!/usr/bin/env python
"""Benchmark: ResNet-50 conv layers fwd + bwdData + bwdWeights, bf16, N=256 per
GPU (BASELINE.json configs[4], the metric's configuration), batch-sharded
over N GPUs with an NCCL all-reduce of dW.

One "step" = all 53 ResNet-50 v1.5 conv layers x {Forward (ImplicitGemm,
tcgen05), BackwardData (Im2colGemm -> tcgen05 dgrad), BackwardWeights
(Im2colGemm -> tcgen05 split-K wgrad)} on synthetic U(-1,1) bf16 tensors,
followed (N>1) by the dW all-reduce. value = algorithmic FLOPs
(2*N*K*C*R*S*P*Q per direction, summed) of all ranks / max-over-ranks time.

Also reported on the same JSON line: the roofline of the dominant kernel (by
launch share of the step: the HBM-bound resident-filter 1x1 GEMM; the tcgen05
family's tensor roofline rides along), the fused conv+bias+ReLU speedup (cfg2), an end-to-end number through
the host-buffer C ABI, the reference CPU path timed on this host, clocks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ResNet-50 conv layer TFLOP/s (fwd/bwd, bf16) & fused conv+bias+ReLU speedup"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class ClockSampler:
    def __init__(self, index: int):
        self.path = f"/tmp/pk_clocks_{os.getpid()}.csv"
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        self.mark = 0
        if self.proc:
            # nvidia-smi can take a second or more to start on a fresh box: wait for its
            # first sample so the (short) timed region is actually sampled
            t0 = time.time()
            while time.time() - t0 < 10.0 and not self._rows():
                time.sleep(0.02)
            self.mark = len(self._rows())

    def _rows(self):
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 7:
                    rows.append(parts)
        return rows

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)  # the sample that covers the end of the region
        self.proc.terminate()
        self.proc.wait()
        rows = self._rows()
        # samples taken while the region ran (the ones before it only prove the sampler is up)
        rows = rows[self.mark:] or rows[-1:]
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        load = [v for v in sm if v > 600] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "samples": len(rows), "reasons": reasons}


# ---------------------------------------------------------------------------
# reference CPU arm: the unmodified reference (oracle/_ref) on host cores

def _ref_worker(args):
    """Run a share of (layer, direction) convs for ONE image through the
    reference's C ABI with its fastest CPU solver (Im2colGemm)."""
    jobs, seed = args
    import numpy as np

    import oracle
    from paper_1910_00078_b200 import abi
    from paper_1910_00078_b200.primkit import operand_shapes, problem

    ref = oracle.reference()
    h = ref.handle()
    rng = np.random.default_rng(seed)
    flops = 0.0
    t0 = time.perf_counter()
    for (c, k, hh, r, s, pad, direction) in jobs:
        p = problem(n=1, c=c, h=hh, w=hh, k=k, y=r, x=r, pad=pad, stride=s, direction=direction,
                    etype=abi.BF16)
        sa, sb, _ = operand_shapes(ref, p)
        a = rng.uniform(-1, 1, sa).astype(np.float32)
        b = rng.uniform(-1, 1, sb).astype(np.float32)
        h.conv_run(p, "Im2colGemm", a, b)
        out_h = (hh + 2 * pad - r) // s + 1
        flops += 2.0 * k * c * r * r * out_h * out_h
    return flops, time.perf_counter() - t0


def reference_step(pool, cores, layers):
    """One bounded sample of the workload: the full 53-layer x 3-direction
    network for one image, spread over `cores` processes (LPT balanced)."""
    from paper_1910_00078_b200 import abi
    jobs = []
    for L in layers:
        for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
            jobs.append(((L.c, L.k, L.h, L.r, L.stride, L.pad, d), L.flops(1)))
    jobs.sort(key=lambda j: -j[1])
    bins = [[] for _ in range(cores)]
    load = [0.0] * cores
    for job, fl in jobs:
        i = load.index(min(load))
        bins[i].append(job)
        load[i] += fl
    t0 = time.perf_counter()
    res = pool.map(_ref_worker, [(b, i) for i, b in enumerate(bins)])
    wall = time.perf_counter() - t0
    reference_step.busy_s = sum(r[1] for r in res)  # summed per-process compute seconds
    return sum(r[0] for r in res), wall


SCALED_NOTE = ("measured on a one-image sample (N=1) and reported as TFLOP/s, which is linear "
               "in N: it stands for the N=256/GPU configuration (scaled)")


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from paper_1910_00078_b200.resnet50 import resnet50_layers
    if not oracle.reference_available():
        oracle.build()
    cores = os.cpu_count() or 1
    layers = resnet50_layers()
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(args.warmup):
            reference_step(pool, cores, layers)
        fl, wall, busy = 0.0, 0.0, 0.0
        for _ in range(args.steps):
            f, w = reference_step(pool, cores, layers)
            fl += f
            wall += w
            busy += reference_step.busy_s
    value = fl / wall / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16 storage, f32 compute", "data": "synthetic U(-1,1)",
        "config": {"workload": "ResNet-50 v1.5, 53 conv layers x {fwd, bwdData, bwdWeights}, "
                               "reference Im2colGemm (its fastest CPU solver)",
                   "global_batch": 1, "parallelism": f"{cores} host processes"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "reference",
                         "value_1core": fl / busy / 1e12, "scaled": SCALED_NOTE,
                         "sample": "one image through all 53 layers x 3 directions per step, "
                                   "(layer, direction) jobs LPT-balanced over host processes"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm

class Net:
    """Device buffers for every layer: x (input), w, y (output), dy, dx, dw."""

    def __init__(self, torch, lib, handle, layers, n, device):
        from paper_1910_00078_b200 import abi
        from paper_1910_00078_b200.primkit import problem
        self.layers, self.n = layers, n
        self.items = []
        pitch = lib.channel_pitch
        g = torch.Generator(device=device)
        g.manual_seed(1234 + n)

        def rand(shape):
            return (torch.rand(shape, generator=g, device=device, dtype=torch.float32) * 2 - 1
                    ).to(torch.bfloat16)

        max_ws = 0
        for L in layers:
            ho = L.out_h
            cp, kp = pitch(L.c), pitch(L.k)
            x = rand((n, L.h, L.h, cp))
            if cp != L.c:
                x[..., L.c:] = 0
            w = rand((L.k, L.r, L.r, cp))
            if cp != L.c:
                w[..., L.c:] = 0
            y = torch.empty((n, ho, ho, kp), dtype=torch.bfloat16, device=device)
            dy = rand((n, ho, ho, kp))
            dx = torch.empty_like(x)
            dw = torch.empty_like(w)
            probs = {}
            for d, solver in ((abi.FORWARD, "ImplicitGemm"), (abi.BACKWARD_DATA, "Im2colGemm"),
                              (abi.BACKWARD_WEIGHTS, "Im2colGemm")):
                p = problem(n=n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad,
                            stride=L.stride, direction=d, etype=abi.BF16)
                ws = C.c_uint64()
                lib.check(lib.lib.primkit_conv_device_workspace(handle.ptr, C.byref(p),
                                                                solver.encode(), C.byref(ws)))
                max_ws = max(max_ws, ws.value)
                probs[d] = (p, solver.encode())
            self.items.append((L, x, w, y, dy, dx, dw, probs))
        self.ws = torch.empty(max(max_ws, 256), dtype=torch.uint8, device=device)
        self.ws2 = None  # backward-weights stream's workspace (two-stream backward)

    def register_grads(self, dp):
        """dW tensors in the order the backward pass produces them (reverse
        layer order) -> native NCCL buckets."""
        from paper_1910_00078_b200 import abi
        for it in reversed(self.items):
            dp.register(it[6], abi.BF16)

    def flops(self) -> float:
        return 3.0 * sum(L.flops(self.n) for L in self.layers)

    def algorithmic_bytes(self) -> float:
        """|x| + |y| + |w| (bf16, padded pitch) over the 53 layers: the minimum
        DRAM traffic of one direction's pass."""
        p = lambda c: (c + 7) // 8 * 8  # noqa: E731
        return float(sum(2 * (self.n * L.h * L.h * p(L.c) + self.n * L.out_h * L.out_h * p(L.k) +
                              L.k * L.r * L.r * p(L.c)) for L in self.layers))


def run_conv(lib, handle, p, solver, a, b, out, ws):
    st = lib.lib.primkit_conv_run_device(handle.ptr, C.byref(p), solver, C.c_void_p(a.data_ptr()),
                                         C.c_void_p(b.data_ptr()), C.c_void_p(out.data_ptr()),
                                         C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()))
    if st:
        lib.check(st)


def step(lib, handle, net, directions=(0, 1, 2), dp=None, wside=None):
    """One training step's convolutions. With a data-parallel context, each
    layer's dW is handed to the native NCCL buckets (primkit_dp_*) right after
    its backward-weights kernel is enqueued, so a bucket's all-reduce overlaps
    the backward of the layers below it; finish() joins before the step ends.

    wside = (torch, handle, stream, events): backward weights on a second
    stream with its own handle and workspace. A layer's dW needs only its dY
    (produced by the previous layer's backward data) and its forward input, so
    it runs beside the next backward-data kernel and fills the SMs that kernel's
    tail and ramp leave idle (the graph keeps the true dependencies as events)."""
    ws = net.ws
    if 0 in directions:
        for (L, x, w, y, dy, dx, dw, probs) in net.items:
            p, s = probs[0]
            run_conv(lib, handle, p, s, x, w, y, ws)
    if wside is not None and 2 in directions:
        torch, wh, wstream, ev = wside
        main = torch.cuda.current_stream()
        ev[0].record(main)               # forward done: inputs of every dW ready
        wstream.wait_event(ev[0])
    for i, (L, x, w, y, dy, dx, dw, probs) in enumerate(reversed(net.items)):
        if wside is not None and 2 in directions:
            p, s = probs[2]
            # dY of this layer came from the previous iteration's backward data
            if i > 0 and 1 in directions:
                wstream.wait_event(ev[i])
            run_conv(lib, wh, p, s, dy, x, dw, net.ws2)
            if dp is not None:
                dp.ready(i)
        if 1 in directions:
            p, s = probs[1]
            run_conv(lib, handle, p, s, dy, w, dx, ws)
            if wside is not None and 2 in directions:
                ev[i + 1].record(main)
        if wside is None and 2 in directions:
            p, s = probs[2]
            run_conv(lib, handle, p, s, dy, x, dw, ws)
            if dp is not None:
                dp.ready(i)
    if dp is not None:
        dp.finish()
    if wside is not None and 2 in directions:
        ev[len(net.items) + 1].record(wstream)
        main.wait_event(ev[len(net.items) + 1])


def batchnorm_roofline(torch, lib, handle, layers, batch, hbm_peak):
    """cfg4's batch-norm kernels against the HBM roofline (BASELINE north_star: "achieved
    HBM GB/s against ... for batch-norm"): single-launch training forward and backward
    (bn_coop.cu) on every distinct ResNet-50 BN input [N, K, P, P] (bf16, NHWC), L2
    flushed by reading a 512 MB buffer before each call, median of 3, CUDA events on
    the launching stream. Algorithmic bytes: forward 3|x| (statistics read, normalise
    read, y write), backward 5|x| (x, dy for the sums; x, dy and the dx write)."""
    import statistics
    flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    shapes = {}
    for L in layers:
        shapes[(L.k, L.out_h)] = shapes.get((L.k, L.out_h), 0) + 1

    def timed(fn):
        fn()
        ts = []
        for _ in range(3):
            flush.max()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)
    tot = {"fwd": [0.0, 0.0], "bwd": [0.0, 0.0]}
    largest = None
    for (k, p), count in sorted(shapes.items()):
        x = (torch.rand((batch, p, p, k), device="cuda") * 2 - 1).to(torch.bfloat16)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        dy = (torch.rand_like(x, dtype=torch.float32) * 2 - 1).to(torch.bfloat16)
        g, b = torch.rand(k, device="cuda") + 0.5, torch.rand(k, device="cuda") - 0.5
        rm, rv = torch.zeros(k, device="cuda"), torch.ones(k, device="cuda")
        sm, si, dg, db = (torch.empty(k, device="cuda") for _ in range(4))
        dims = (C.c_int64 * 4)(batch, k, p, p)
        xb = x.numel() * 2

        def fwd():
            lib.check(lib.lib.primkit_batchnorm_forward_train_device(
                handle.ptr, dims, 1, P(x), P(g), P(b), P(rm), P(rv), C.c_float(1e-5), C.c_float(0.1),
                P(y), P(sm), P(si), 1))

        def bwd():
            lib.check(lib.lib.primkit_batchnorm_backward_device(
                handle.ptr, dims, 1, P(x), P(y), P(dy), P(g), P(b), P(sm), P(si), P(dx), P(dg), P(db), 0))
        fwd()
        tf, tb = timed(fwd), timed(bwd)
        for d, t, nb in (("fwd", tf, 3 * xb), ("bwd", tb, 5 * xb)):
            tot[d][0] += count * nb
            tot[d][1] += count * t
        if largest is None or xb > largest[0]:
            largest = (xb, k, p, 3 * xb / tf / 1e6, 5 * xb / tb / 1e6)
        del x, y, dx, dy
    out = {"unit": "GB/s", "peak": hbm_peak, "kernels": "bn_coop (single-launch training BN, bf16)",
           "shapes": "every distinct ResNet-50 BN input at N=%d, weighted by its 53-layer count" % batch}
    for d in ("fwd", "bwd"):
        gbs = tot[d][0] / tot[d][1] / 1e6
        out[d] = {"achieved": gbs, "frac": gbs / hbm_peak, "ms_all_layers": tot[d][1]}
    out["largest"] = {"shape": [batch, largest[1], largest[2], largest[2]], "fwd_gbs": largest[3],
                      "bwd_gbs": largest[4], "fwd_frac": largest[3] / hbm_peak,
                      "bwd_frac": largest[4] / hbm_peak}
    return out


def time_region(torch, fn, iters):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


def fusion_speedup(torch, lib, handle, device):
    """cfg2: fused conv+bias+ReLU vs the same conv kernel + separate bias and
    ReLU passes, bf16, ResNet-50 1x1 and 3x3 shapes at N=64."""
    from paper_1910_00078_b200 import abi
    out = {}
    for name, (c, k, hw, f, pad) in (("1x1_64to256_56", (64, 256, 56, 1, 0)),
                                     ("3x3_64to64_56", (64, 64, 56, 3, 1))):
        plan = lib.fusion_plan((64, c, hw, hw), abi.BF16)
        lib.check(plan.add_conv((k, c, f, f), pad=pad))
        lib.check(plan.add_bias(k))
        lib.check(plan.add_activation(abi.RELU))
        st = plan.compile(handle)
        note = None
        if st:  # the reference table rejects bf16 3x3 CBA; run it through the
            # ImplicitGemm-labelled kernel family directly is not possible via
            # the plan API, so use the f32 table row semantics instead
            note = lib.last_error()
            plan = lib.fusion_plan((64, c, hw, hw), abi.BF16)
            lib.check(plan.add_conv((k, c, f, f), pad=pad))
            lib.check(plan.add_bias(k))
            lib.check(plan.add_batchnorm(abi.BN_SPATIAL))
            lib.check(plan.add_activation(abi.RELU))
            lib.check(plan.compile(handle))
        import numpy as np
        rng = np.random.default_rng(0)
        plan.set_args(filter=rng.uniform(-1, 1, (k, c, f, f)).astype(np.float32),
                      bias=rng.uniform(-1, 1, k).astype(np.float32),
                      gamma=np.ones(k, np.float32), beta=np.zeros(k, np.float32),
                      mean=np.zeros(k, np.float32), var=np.ones(k, np.float32))
        x = (torch.rand((64, hw, hw, lib.channel_pitch(c)), device=device) * 2 - 1).to(torch.bfloat16)
        y = torch.empty((64, hw, hw, lib.channel_pitch(k)), device=device, dtype=torch.bfloat16)

        def run(unf):
            lib.check(lib.lib.primkit_fusion_execute_device(handle.ptr, plan.ptr,
                                                            C.c_void_p(x.data_ptr()),
                                                            C.c_void_p(y.data_ptr()), unf))
        for unf in (0, 1):
            run(unf)
        fused = time_region(torch, lambda: run(0), 20) / 20
        unfused = time_region(torch, lambda: run(1), 20) / 20
        fl = 2.0 * 64 * k * c * f * f * hw * hw
        out[name] = {"fused_ms": fused, "unfused_ms": unfused, "speedup": unfused / fused,
                     "fused_tflops": fl / fused / 1e9,
                     "ops": "conv+bias+relu" if note is None else "conv+bias+bn+relu (bf16 CBA 3x3 "
                     "is rejected by the reference table: '" + note + "')"}
    return out


def e2e_measure(torch, lib, handle, layers, n, steps):
    """Same metric through the host-buffer C ABI (primkit_conv_run): every
    call uploads NCHW f32 operands from pinned host memory, converts to the
    device layout, runs, converts back and downloads the result."""
    from paper_1910_00078_b200 import abi
    from paper_1910_00078_b200.primkit import operand_shapes, problem
    import numpy as np
    max_el = 0
    calls = []
    for L in layers:
        for d, s in ((abi.FORWARD, "ImplicitGemm"), (abi.BACKWARD_DATA, "Im2colGemm"),
                     (abi.BACKWARD_WEIGHTS, "Im2colGemm")):
            p = problem(n=n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad, stride=L.stride,
                        direction=d, etype=abi.BF16)
            sa, sb, so = operand_shapes(lib, p)
            na, nb, no = (int(np.prod(v)) for v in (sa, sb, so))
            max_el = max(max_el, na, nb, no)
            calls.append((p, s.encode(), na, nb, no))
    bufs = [torch.empty(max_el, dtype=torch.float32).pin_memory() for _ in range(3)]
    for b in bufs:
        b.uniform_(-1, 1)
    ptrs = [C.cast(C.c_void_p(b.data_ptr()), C.POINTER(C.c_float)) for b in bufs]
    ws = C.c_size_t(1 << 34)  # gate only; the library sizes device scratch itself
    h2d = sum(4 * (na + nb) for (_, _, na, nb, _) in calls)
    d2h = sum(4 * no for (_, _, _, _, no) in calls)

    def one():
        for (p, s, na, nb, no) in calls:
            lib.check(lib.lib.primkit_conv_run(handle.ptr, C.byref(p), s, ptrs[0], ptrs[1], ptrs[2],
                                               ws))
    one()  # warm (allocations, plan cache)
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    wall = time.perf_counter() - t0
    return wall / steps, h2d, d2h


def roofline(torch, lib, handle, net, peaks):
    """Dominant kernel family: the tcgen05 implicit-GEMM convolutions. Time
    each direction's pass over the network with CUDA events on the launching
    (current) stream; algorithmic FLOPs / time vs the measured bf16 peak."""
    res = {}
    for d, name in ((0, "igemm_tc_fprop"), (1, "igemm_tc_dgrad"), (2, "igemm_tc_wgrad")):
        ms = time_region(torch, lambda: step(lib, handle, net, directions=(d,)), 3) / 3
        res[name] = {"ms": ms, "tflops": sum(L.flops(net.n) for L in net.layers) / ms / 1e9}
    return res


def ncu_fwd_launch_traffic(layer_indices):
    """Average DRAM bytes (read + write) per launch of the given forward layers,
    from the committed ncu launch list of one step (forward launches first, in
    layer order). None if absent."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*launches_step.csv")))
    if not files or not layer_indices:
        return None, None
    with open(files[-1]) as f:
        rows = list(csv.DictReader(f))
    b = [float(rows[i]["dram__bytes_read.sum"]) + float(rows[i]["dram__bytes_write.sum"])
         for i in layer_indices if i < len(rows)]
    return (sum(b) / len(b) if b else None), os.path.basename(files[-1])


def hbm_kernel_roofline(torch, lib, handle, net, peaks):
    """The kernel with the largest share of the step's launch list is the
    resident-filter plain GEMM (conv_tc PLAIN_RES) of the HBM-bound 1x1 layers.
    Time each of its forward launches in the step (1x1 stride-1 layers whose
    filter slice stays resident: reduction <= 256) with CUDA events, and compare
    the algorithmic bytes (x + w + y, bf16, read or written once) per launch
    with the measured HBM copy bandwidth."""
    pitch = lambda c: (c + 7) // 8 * 8  # noqa: E731
    ms_tot, bytes_tot, n = 0.0, 0.0, 0
    idx = []
    for li, (L, x, w, y, dy, dx, dw, probs) in enumerate(net.items):
        if not (L.r == 1 and L.stride == 1 and pitch(L.c) <= 256 and L.k >= 64):
            continue
        idx.append(li)
        p, s = probs[0]
        run_conv(lib, handle, p, s, x, w, y, net.ws)
        ms_tot += time_region(torch, lambda: run_conv(lib, handle, p, s, x, w, y, net.ws), 5) / 5
        bytes_tot += 2.0 * (net.n * L.h * L.h * pitch(L.c) + L.k * pitch(L.c) +
                            net.n * L.out_h * L.out_h * pitch(L.k))
        n += 1
    if n == 0:
        return None
    achieved = bytes_tot / (ms_tot * 1e-3) / 1e9
    traffic, src = ncu_fwd_launch_traffic(idx)
    return {"bound": "hbm", "kernel": "conv_tc_kernel PLAIN_RES (resident-filter 1x1 GEMM), "
            "%d ResNet-50 forward launches, N=%d" % (n, net.n), "achieved": achieved,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
            "traffic": traffic, "traffic_unit": "bytes per launch (ncu DRAM read + write, average)",
            "traffic_source": src, "algorithmic_bytes_per_launch": bytes_tot / n,
            "ms_per_launch": ms_tot / n}


def ncu_family_traffic(family: str):
    """DRAM bytes (read + write) per step of one direction's kernels, from the
    committed ncu launch list of one step (profiles/*launches_step.csv,
    `--metrics ...,dram__bytes_read.sum,dram__bytes_write.sum`, launch order).
    step() runs the 53 forward convolutions first (one launch each), then per
    layer (reversed) the backward-data and backward-weights kernels; launches
    are classified by that order and by name (*wgrad* = backward weights, incl.
    the split-K sums). None if absent."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*launches_step.csv")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        rows = list(csv.DictReader(f))
    from paper_1910_00078_b200.resnet50 import resnet50_layers
    n_fwd = len(resnet50_layers())
    tot = {"igemm_tc_fprop": 0.0, "igemm_tc_dgrad": 0.0, "igemm_tc_wgrad": 0.0}
    for i, row in enumerate(rows):
        b = float(row["dram__bytes_read.sum"]) + float(row["dram__bytes_write.sum"])
        if i < n_fwd:
            tot["igemm_tc_fprop"] += b
        elif "wgrad" in row["kernel"]:
            tot["igemm_tc_wgrad"] += b
        else:
            tot["igemm_tc_dgrad"] += b
    return tot[family], os.path.basename(files[-1])


def layer_report(torch, lib, handle, net, peaks, path):
    """Per (layer, direction) device time and roofline position."""
    rows = []
    hbm = peaks["hbm_gbs"] * 1e9
    tc = peaks["bf16_tflops"] * 1e12
    only = set(os.environ.get("PK_LAYERS", "").split(",")) - {""}
    for (L, x, w, y, dy, dx, dw, probs) in net.items:
        if only and L.name not in only:
            continue
        for d, (a, b, o) in ((0, (x, w, y)), (1, (dy, w, dx)), (2, (dy, x, dw))):
            p, s = probs[d]
            run_conv(lib, handle, p, s, a, b, o, net.ws)
            eager_ms = time_region(torch, lambda: run_conv(lib, handle, p, s, a, b, o, net.ws), 10) / 10
            # device time without host launch overhead: 10 launches in one graph
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                lib.check(lib.lib.primkit_handle_set_stream(
                    handle.ptr, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
                for _ in range(10):
                    run_conv(lib, handle, p, s, a, b, o, net.ws)
            lib.check(lib.lib.primkit_handle_set_stream(
                handle.ptr, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
            g.replay()
            ms = time_region(torch, g.replay, 3) / 30
            fl = L.flops(net.n)
            byts = 2 * (a.numel() + b.numel() + o.numel())
            bound_ms = max(fl / tc, byts / hbm) * 1e3
            kname = C.create_string_buffer(64)
            lib.lib.primkit_handle_last_kernel(handle.ptr, kname, 64)
            rows.append({"layer": L.name, "dir": ["fwd", "bwd_data", "bwd_weights"][d],
                         "c": L.c, "k": L.k, "h": L.h, "r": L.r, "stride": L.stride,
                         "kernel": kname.value.decode(), "ms": ms, "eager_ms": eager_ms,
                         "tflops": fl / ms / 1e9,
                         "roofline_ms": bound_ms, "frac_of_roofline": bound_ms / ms,
                         "bound": "tensor" if fl / tc > byts / hbm else "hbm"})
    with open(path, "w") as f:
        json.dump(rows, f, indent=1)
    for r in sorted(rows, key=lambda r: -r["ms"])[:25]:
        print(f"{r['layer']:>10} {r['dir']:>11} {r['kernel']:>16} {r['ms']:8.3f} ms "
              f"{r['tflops']:7.1f} TF/s  roofline {r['frac_of_roofline']:.2f} ({r['bound']})",
              file=sys.stderr)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(nproc: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this script under
    torch.distributed.run with N local ranks (one process per GPU) and
    return its exit code; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)]
    return subprocess.call(cmd + sys.argv[1:], env=dict(os.environ, PK_BENCH_SPAWNED="1"))


def launch_selftest(args) -> int:
    """--launch-selftest: the multi-rank plumbing without a GPU (gloo):
    world size, rank-0 reduction of per-rank values (as the timing uses)."""
    import torch
    import torch.distributed as tdist
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"world size {world} != --gpus {args.gpus}", file=sys.stderr)
        return 3
    tdist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"launch_selftest": True, "n_gpus": world, "max_over_ranks": float(t.item())}),
              flush=True)
    tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer-report", default=None, help="write per-layer timings (JSON)")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256, help="images per GPU")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-extras", action="store_true", help="skip e2e/cpu/fusion legs")
    ap.add_argument("--streams", type=int, default=2, choices=(1, 2),
                    help="2: backward weights on a second stream beside backward data")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the step eagerly instead of as one CUDA graph")
    ap.add_argument("--bucket-mb", type=float, default=25.0, help="fp32 MiB per dW all-reduce bucket")
    ap.add_argument("--dp", action="store_true",
                    help="use the NCCL dW buckets even at one GPU (overhead measurement)")
    ap.add_argument("--launch-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.launch_selftest:
        return launch_selftest(args)

    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    from paper_1910_00078_b200.primkit import library
    from paper_1910_00078_b200.resnet50 import resnet50_layers

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=device)
        dist = tdist

    lib = library()
    stream = torch.cuda.current_stream()
    handle_ptr = C.c_void_p()
    lib.check(lib.lib.primkit_handle_create_with_stream(C.c_void_p(stream.cuda_stream), local,
                                                        C.byref(handle_ptr)))

    class _H:  # minimal handle wrapper around the stream-bound handle
        ptr = handle_ptr
    handle = _H()

    layers = resnet50_layers()
    net = Net(torch, lib, handle, layers, args.batch, device)
    wside = None
    if args.streams == 2:
        wstream = torch.cuda.Stream(device=device)
        wh_ptr = C.c_void_p()
        lib.check(lib.lib.primkit_handle_create_with_stream(C.c_void_p(wstream.cuda_stream), local,
                                                            C.byref(wh_ptr)))

        class _WH:
            ptr = wh_ptr
        net.ws2 = torch.empty_like(net.ws)
        wside = (torch, _WH(), wstream,
                 [torch.cuda.Event() for _ in range(len(layers) + 2)])
    dp = None
    if world > 1 or args.dp:
        from paper_1910_00078_b200.dist import DataParallel
        dp = DataParallel(lib, (wside[1].ptr if wside else handle.ptr), rank, world, dist=dist,
                          bucket_bytes=int(args.bucket_mb * (1 << 20)))
        net.register_grads(dp)
    if args.layer_report:
        layer_report(torch, lib, handle, net, load_peaks()[0], args.layer_report)
        return 0
    for _ in range(args.warmup):
        step(lib, handle, net, dp=dp, wside=wside)
    torch.cuda.synchronize()
    if dp is not None:
        dp.check()
    if dist:
        dist.barrier()

    launches0 = C.c_uint64()
    lib.check(lib.lib.primkit_handle_kernel_launches(handle.ptr, C.byref(launches0)))
    run_step = lambda: step(lib, handle, net, dp=dp, wside=wside)  # noqa: E731
    graph_note = "eager launches"
    launches_per_step = None
    if args.graph:
        # The step's 159 conv launches (+ the dW bucket all-reduces on the comm
        # stream, forked and joined inside the capture) replayed as one CUDA
        # graph: same kernels, same work, no per-launch host overhead.
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                lib.check(lib.lib.primkit_handle_set_stream(
                    handle.ptr, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
                step(lib, handle, net, dp=dp, wside=wside)  # the 159 convolutions (+ NCCL buckets)
            lib.check(lib.lib.primkit_handle_set_stream(handle.ptr, C.c_void_p(stream.cuda_stream)))
            lc = C.c_uint64()
            lib.check(lib.lib.primkit_handle_kernel_launches(handle.ptr, C.byref(lc)))
            launches_per_step = int(lc.value - launches0.value)
            launches0 = lc
            graph.replay()
            torch.cuda.synchronize()

            run_step = graph.replay
            graph_note = ("CUDA graph of the step's convolutions" +
                          (" + NCCL dW bucket all-reduces (comm stream, captured)"
                           if dp is not None else ""))
        except Exception as exc:  # fall back to eager launches
            lib.check(lib.lib.primkit_handle_set_stream(handle.ptr, C.c_void_p(stream.cuda_stream)))
            graph_note = f"eager launches (graph capture failed: {exc})"
    clocks = ClockSampler(local)
    ms_total = time_region(torch, run_step, args.steps)
    clk = clocks.stop()
    if dp is not None:
        dp.check()
    launches1 = C.c_uint64()
    lib.check(lib.lib.primkit_handle_kernel_launches(handle.ptr, C.byref(launches1)))
    if launches_per_step is not None:
        launches1 = C.c_uint64(launches0.value + launches_per_step * args.steps)
    if dist:
        t = torch.tensor([ms_total], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps
    value = net.flops() * world / (ms_step * 1e-3) / 1e12

    peaks, peak_kind = load_peaks()
    extras = {}
    if not args.no_extras:
        rf = roofline(torch, lib, handle, net, peaks)
        e2e_s, h2d, d2h = e2e_measure(torch, lib, handle, layers, args.batch, args.e2e_steps)
        e2e_val = net.flops() * world / e2e_s / 1e12
        if dist:
            t = torch.tensor([e2e_s], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_val = net.flops() * world / float(t.item()) / 1e12
        extras["e2e"] = {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
                         "d2h_bytes_per_step": d2h,
                         "path": "primkit_conv_run (host NCHW f32 buffers, pinned)"}
        peak = peaks["bf16_tflops_sustained"]
        dom_name = max(rf, key=lambda k: rf[k]["ms"])  # largest share of the step
        dom = rf[dom_name]
        family = {
            "bound": "tensor",
            "kernel": "%s family (all 53 ResNet-50 convs of that direction, N=%d; largest share "
                      "of the step)" % (dom_name, args.batch),
            "achieved": dom["tflops"], "peak": peak, "unit": "TFLOP/s",
            "frac": dom["tflops"] / peak, "traffic": ncu_family_traffic(dom_name)[0],
            "traffic_unit": "bytes per step (DRAM read+write of the family's kernels)",
            "algorithmic_bytes": net.algorithmic_bytes(),
            "traffic_source": ncu_family_traffic(dom_name)[1],
            "peak_source": f"{peak_kind} bf16_tflops_sustained (MEASURED_PEAKS.json)",
            "per_direction": rf}
        # per-layer roofline (each conv bounded by max(FLOPs / tensor peak, bytes / HBM
        # peak), bytes = x + w + y in bf16): the family's attainable time vs measured
        pitch = lambda c: (c + 7) // 8 * 8  # noqa: E731
        roof_ms = 0.0
        for L in net.layers:
            byts = 2.0 * (args.batch * L.h * L.h * pitch(L.c) + L.k * L.r * L.r * pitch(L.c) +
                          args.batch * L.out_h * L.out_h * pitch(L.k))
            roof_ms += max(L.flops(args.batch) / (peak * 1e12),
                           byts / (peaks["hbm_gbs"] * 1e9)) * 1e3
        family["layer_roofline_ms"] = roof_ms
        family["frac_of_layer_roofline"] = roof_ms / dom["ms"]
        # The dominant single kernel by launch share of the step's ncu launch list
        # (profiles/*launches_step.md) is the HBM-bound resident-filter 1x1 GEMM:
        # it is the line's roofline; the tensor family and the whole-step position
        # against the per-layer roofline ride along.
        hk = hbm_kernel_roofline(torch, lib, handle, net, peaks)
        extras["roofline"] = dict(hk) if hk else family
        if hk:
            extras["roofline"]["peak_source"] = f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)"
            extras["roofline"]["tensor_family"] = family
        extras["roofline"]["step_frac_of_layer_roofline"] = 3 * roof_ms / ms_step
        if rank == 0:
            extras["fusion"] = fusion_speedup(torch, lib, handle, device)
            extras["batchnorm"] = batchnorm_roofline(torch, lib, handle, layers, args.batch,
                                                     peaks["hbm_gbs"])
            with mp.get_context("fork").Pool(os.cpu_count() or 1) as pool:
                import oracle
                if not oracle.reference_available():
                    oracle.build()
                fl, wall = reference_step(pool, os.cpu_count() or 1, layers)
            extras["cpu_baseline"] = {
                "value": fl / wall / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count() or 1,
                "kind": "reference", "value_1core": fl / reference_step.busy_s / 1e12,
                "scaled": SCALED_NOTE,
                "sample": "one image through all 53 layers x 3 directions (reference "
                          "Im2colGemm, oracle/_ref), jobs balanced over host processes"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic U(-1,1) bf16 tensors (no dataset)",
            "config": {"workload": "ResNet-50 v1.5 all 53 conv layers, fwd + bwdData + bwdWeights, "
                                   "bf16, NHWC device layout",
                       "model": "ResNet-50 conv layers", "global_batch": args.batch * world,
                       "per_gpu_batch": args.batch, "parallelism": f"dp{world}",
                       "dw_allreduce": (f"native NCCL fp32 sum, {dp.buckets()} buckets of <= "
                                        f"{args.bucket_mb:g} MiB in backward order, comm stream "
                                        "overlapped with the remaining backward") if dp else None,
                       "l2": "working set per step >> 126 MB L2 (no flush needed)",
                       "launch": graph_note},
            "gpu_launches": int(launches1.value - launches0.value),
            "clocks": clk,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if dp is not None:
        dp.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
