#!/usr/bin/env python
"""Per-config measurements for BASELINE.json configs[0..3] (configs[4], the
full ResNet-50 step, is bench.py). Writes one JSON document (stdout or
--out) with device times from CUDA events (median of --iters after warm-up),
TFLOP/s, fusion speedups, Find's selection and the reference CPU time where
it is bounded (cfg1).

  cfg1  fp32 3x3 fwd N=8 C=K=64 56x56 (Direct SIMT; other fp32 solvers beside)
  cfg2  fused conv+bias+ReLU (fp32 and bf16) vs the unfused op sequence,
        ResNet-50 1x1 (64->256) and 3x3 (64->64) at N=64
  cfg3  VGG-16 3x3 layers bf16 N=128: Winograd F(2,3) vs implicit GEMM, and
        the Find protocol's choice (device-timed, reduced N)
  cfg4  ResNet-50 conv + training BN (+ReLU), bf16 N=256, fused statistics
        epilogues (fwd and bwd) vs conv + standalone BN

    python tools/bench_configs.py [--only cfg1,cfg3] [--iters 5] [--out f.json]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import library, operand_shapes, problem  # noqa: E402
from paper_1910_00078_b200.resnet50 import resnet50_layers  # noqa: E402

VGG16 = [(3, 64, 224), (64, 64, 224), (64, 128, 112), (128, 128, 112), (128, 256, 56),
         (256, 256, 56), (256, 256, 56), (256, 512, 28), (512, 512, 28), (512, 512, 28),
         (512, 512, 14), (512, 512, 14), (512, 512, 14)]


def vp(t):
    return C.c_void_p(t.data_ptr())


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


class Dev:
    """Device handle bound to torch's current stream + tensor helpers."""

    def __init__(self):
        self.lib = library()
        self.h = C.c_void_p()
        self.lib.check(self.lib.lib.primkit_handle_create_with_stream(
            C.c_void_p(torch.cuda.current_stream().cuda_stream), 0, C.byref(self.h)))

    def act(self, n, h, w, c, dtype):
        p = self.lib.channel_pitch(c)
        t = (torch.rand((n, h, w, p), device="cuda") * 2 - 1).to(dtype)
        if p != c:
            t[..., c:] = 0
        return t

    def ws(self, p, solver, fn="primkit_conv_device_workspace"):
        b = C.c_uint64()
        self.lib.check(getattr(self.lib.lib, fn)(self.h, C.byref(p), solver, C.byref(b)))
        return torch.empty(max(b.value, 256), dtype=torch.uint8, device="cuda")

    def conv(self, p, solver, a, b, o, ws):
        self.lib.check(self.lib.lib.primkit_conv_run_device(self.h, C.byref(p), solver, vp(a), vp(b),
                                                            vp(o), vp(ws), C.c_size_t(ws.numel())))

    def last_kernel(self):
        buf = C.create_string_buffer(96)
        self.lib.lib.primkit_handle_last_kernel(self.h, buf, 96)
        return buf.value.decode()


def flops(p, ho, wo):
    return 2.0 * p.n * p.k * (p.c // p.groups) * p.y * p.x * ho * wo


def cfg1(d, iters):
    p = problem(n=8, c=64, h=56, w=56, k=64, y=3, x=3, pad=1)
    x, w = d.act(8, 56, 56, 64, torch.float32), d.act(64, 3, 3, 64, torch.float32)
    y = torch.empty((8, 56, 56, 64), device="cuda")
    out = {"problem": "fp32 3x3 fwd N=8 C=K=64 56x56 pad1", "gflop": flops(p, 56, 56) / 1e9}
    for s in ("Direct", "Im2colGemm", "ImplicitGemm", "Winograd"):
        ws = d.ws(p, s.encode())
        ms = timed(lambda: d.conv(p, s.encode(), x, w, y, ws), iters)
        out[s] = {"ms": ms, "tflops": out["gflop"] / ms, "kernel": d.last_kernel()}
    # the reference's own CPU Direct on the same problem (one host core)
    import oracle
    if not oracle.reference_available():
        oracle.build()
    ref = oracle.reference()
    rh = ref.handle()
    rng = np.random.default_rng(1)
    sa, sb, _ = operand_shapes(ref, p)
    a = rng.uniform(-1, 1, sa).astype(np.float32)
    b = rng.uniform(-1, 1, sb).astype(np.float32)
    t0 = time.perf_counter()
    rh.conv_run(p, "Direct", a, b)
    cpu = (time.perf_counter() - t0) * 1e3
    out["reference_cpu_direct"] = {"ms": cpu, "cores": 1, "tflops": out["gflop"] / cpu}
    out["speedup_vs_reference_direct"] = cpu / out["Direct"]["ms"]
    return out


def cfg2(d, iters):
    out = {}
    for et, name in ((abi.F32, "f32"), (abi.BF16, "bf16")):
        tdt = torch.float32 if et == abi.F32 else torch.bfloat16
        for tag, (c, k, hw, f, pad, algo) in (("1x1_64to256_56", (64, 256, 56, 1, 0, "Direct")),
                                              ("3x3_64to64_56", (64, 64, 56, 3, 1, "Winograd"))):
            lib = d.lib
            plan = lib.fusion_plan((64, c, hw, hw), et)
            lib.check(plan.add_conv((k, c, f, f), pad=pad, algo=algo))
            lib.check(plan.add_bias(k))
            lib.check(plan.add_activation(abi.RELU))
            st = plan.compile(_H(d.h))
            entry = {"ops": "conv+bias+relu", "label": algo}
            if st:
                # table rejects this row (e.g. bf16 3x3 CBA): run CBNA instead
                entry["table_verdict"] = lib.last_error()
                plan = lib.fusion_plan((64, c, hw, hw), et)
                lib.check(plan.add_conv((k, c, f, f), pad=pad, algo="Direct"))
                lib.check(plan.add_bias(k))
                lib.check(plan.add_batchnorm(abi.BN_SPATIAL))
                lib.check(plan.add_activation(abi.RELU))
                lib.check(plan.compile(_H(d.h)))
                entry["ops"] = "conv+bias+bn+relu"
            rng = np.random.default_rng(0)
            plan.set_args(filter=rng.uniform(-1, 1, (k, c, f, f)).astype(np.float32),
                          bias=rng.uniform(-1, 1, k).astype(np.float32),
                          gamma=np.ones(k, np.float32), beta=np.zeros(k, np.float32),
                          mean=np.zeros(k, np.float32), var=np.ones(k, np.float32))
            x = d.act(64, hw, hw, c, tdt)
            y = torch.empty((64, hw, hw, lib.channel_pitch(k)), device="cuda", dtype=tdt)

            def run(unf):
                lib.check(lib.lib.primkit_fusion_execute_device(d.h, plan.ptr, vp(x), vp(y), unf))
            fused = timed(lambda: run(0), iters)
            kern = d.last_kernel()
            unfused = timed(lambda: run(1), iters)
            p = problem(n=64, c=c, h=hw, w=hw, k=k, y=f, x=f, pad=pad)
            entry.update({"fused_ms": fused, "unfused_ms": unfused, "speedup": unfused / fused,
                          "fused_tflops": flops(p, hw, hw) / fused / 1e9, "kernel": kern})
            out[f"{name}_{tag}"] = entry
    return out


class _H:
    def __init__(self, ptr):
        self.ptr = ptr


def cfg3(d, iters, n=128):
    rows, tot = [], {"ImplicitGemm": 0.0, "Winograd": 0.0}
    fl_total = 0.0
    for (c, k, hw) in VGG16:
        p = problem(n=n, c=c, h=hw, w=hw, k=k, y=3, x=3, pad=1, etype=abi.BF16)
        x, w = d.act(n, hw, hw, c, torch.bfloat16), d.act(k, 3, 3, c, torch.bfloat16)
        y = torch.empty((n, hw, hw, d.lib.channel_pitch(k)), device="cuda", dtype=torch.bfloat16)
        fl = flops(p, hw, hw)
        fl_total += fl
        row = {"layer": f"{c}->{k}@{hw}", "gflop": fl / 1e9}
        for s in ("ImplicitGemm", "Winograd", "Winograd-F43"):
            solver = s.split("-")[0].encode()
            os.environ["PK_WINOGRAD_M"] = "4" if s.endswith("F43") else "2"
            ws = d.ws(p, solver)
            ms = timed(lambda: d.conv(p, solver, x, w, y, ws), iters)
            row[s] = {"ms": ms, "tflops": fl / ms / 1e9, "kernel": d.last_kernel()}
            tot[s] = tot.get(s, 0.0) + ms
        os.environ.pop("PK_WINOGRAD_M", None)
        # Find (device-timed, every applicable solver) on a reduced batch
        pf = problem(n=2, c=c, h=hw, w=hw, k=k, y=3, x=3, pad=1, etype=abi.BF16)
        hf = d.lib.handle()
        rng = np.random.default_rng(3)
        sa, sb, _ = operand_shapes(d.lib, pf)
        found, _ = hf.find(pf, rng.uniform(-1, 1, sa).astype(np.float32),
                           rng.uniform(-1, 1, sb).astype(np.float32), 1 << 34, 8)
        row["find_n2"] = [(r.solver_name.decode() if isinstance(r.solver_name, bytes) else
                           str(r.solver_name), round(r.time_ms, 4)) for r in found]
        rows.append(row)
    return {"batch": n, "layers": rows,
            "total_ms": tot, "tflops": {s: fl_total / v / 1e9 for s, v in tot.items()},
            "note": "Winograd F(2,3)/F(4,3) (tensor-core, bf16) effective TFLOP/s use the direct-conv flop count"}


def cfg4(d, iters, n=256):
    lib = d.lib
    out = {"fwd": {"fused_ms": 0.0, "unfused_ms": 0.0}, "bwd": {"fused_ms": 0.0, "unfused_ms": 0.0}}
    layers = resnet50_layers()
    for L in layers:
        ho = L.out_h
        p = problem(n=n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad, stride=L.stride,
                    etype=abi.BF16)
        x, w = d.act(n, L.h, L.h, L.c, torch.bfloat16), d.act(L.k, L.r, L.r, L.c, torch.bfloat16)
        kp = lib.channel_pitch(L.k)
        conv = torch.empty((n, ho, ho, kp), device="cuda", dtype=torch.bfloat16)
        z = torch.empty_like(conv)
        vec = lambda v: torch.full((L.k,), v, device="cuda")  # noqa: E731
        g, b, rm, rv, sm, si = vec(1.0), vec(0.0), vec(0.0), vec(1.0), vec(0.0), vec(1.0)
        ws = d.ws(p, b"ImplicitGemm", "primkit_conv_bn_workspace")

        def fused():
            lib.check(lib.lib.primkit_conv_bn_forward_train_device(
                d.h, C.byref(p), b"ImplicitGemm", vp(x), vp(w), vp(g), vp(b), vp(rm), vp(rv),
                C.c_float(1e-5), C.c_float(0.1), vp(conv), vp(z), vp(sm), vp(si), 1, vp(ws),
                C.c_size_t(ws.numel())))
        dims = (C.c_int64 * 4)(n, L.k, ho, ho)

        def unfused():
            d.conv(p, b"ImplicitGemm", x, w, conv, ws)
            lib.check(lib.lib.primkit_batchnorm_forward_train_device(
                d.h, dims, abi.BF16, vp(conv), vp(g), vp(b), vp(rm), vp(rv), C.c_float(1e-5),
                C.c_float(0.1), vp(z), vp(sm), vp(si), 1))
        tf, tu = timed(fused, iters), timed(unfused, iters)
        out["fwd"]["fused_ms"] += tf
        out["fwd"]["unfused_ms"] += tu
        kname = C.create_string_buffer(96)
        fused()
        lib.lib.primkit_handle_last_kernel(d.h, kname, 96)
        out.setdefault("layers", []).append({"layer": L.name, "fwd_fused_ms": tf, "fwd_unfused_ms": tu,
                                             "fwd_kernel": kname.value.decode()})
        # backward: this layer's dgrad produces dz of the preceding BN (C channels)
        if L.c % 8 == 0 and L.c >= 64:
            pb = problem(n=n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad, stride=L.stride,
                         direction=abi.BACKWARD_DATA, etype=abi.BF16)
            dy = d.act(n, ho, ho, L.k, torch.bfloat16)
            dz = torch.empty_like(x)
            bnx, bdx, bny = d.act(n, L.h, L.h, L.c, torch.bfloat16), torch.empty_like(x), torch.empty_like(x)
            vc = lambda v: torch.full((L.c,), v, device="cuda")  # noqa: E731
            gc, bc, mc, ic, dg, db = vc(1.0), vc(0.0), vc(0.0), vc(1.0), vc(0.0), vc(0.0)
            wsb = d.ws(pb, b"Im2colGemm", "primkit_conv_bn_workspace")

            def bfused():
                lib.check(lib.lib.primkit_conv_backward_data_bn_device(
                    d.h, C.byref(pb), b"Im2colGemm", vp(dy), vp(w), vp(dz), vp(bnx), vp(gc), vp(bc),
                    vp(mc), vp(ic), 1, vp(bdx), vp(dg), vp(db), vp(wsb), C.c_size_t(wsb.numel())))
            dimc = (C.c_int64 * 4)(n, L.c, L.h, L.h)

            def bunfused():
                d.conv(pb, b"Im2colGemm", dy, w, dz, wsb)
                lib.check(lib.lib.primkit_batchnorm_backward_device(
                    d.h, dimc, abi.BF16, vp(bnx), vp(bny), vp(dz), vp(gc), vp(bc), vp(mc), vp(ic),
                    vp(bdx), vp(dg), vp(db), 1))
            tbf, tbu = timed(bfused, iters), timed(bunfused, iters)
            out["bwd"]["fused_ms"] += tbf
            out["bwd"]["unfused_ms"] += tbu
            out["layers"][-1].update({"bwd_fused_ms": tbf, "bwd_unfused_ms": tbu})
    for k in ("fwd", "bwd"):
        out[k]["speedup"] = out[k]["unfused_ms"] / out[k]["fused_ms"]
    out["batch"] = n
    out["note"] = ("fwd: conv + BN-train + ReLU for all 53 layers (fused: statistics in the conv "
                   "epilogue + one normalise pass); bwd: dgrad producing each BN's dz + BN backward "
                   "(fused: reductions in the dgrad epilogue + one dx pass), unfused = conv + "
                   "standalone two-pass BN. bwd unfused passes the BN output for the ReLU mask.")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg2,cfg3,cfg4")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    d = Dev()
    res = {}
    for name in a.only.split(","):
        t0 = time.time()
        res[name] = globals()[name](d, a.iters)
        res[name]["wall_s"] = time.time() - t0
        print(name, "done", file=sys.stderr, flush=True)
    text = json.dumps(res, indent=1, default=str)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    print(text)


if __name__ == "__main__":
    main()
