"""Parity at the benchmarked configurations (BASELINE.json configs[0..4]).

* Every (layer, direction) problem of bench.py's step — the 53 ResNet-50 v1.5
  convolutions x {Forward/ImplicitGemm, BackwardData/Im2colGemm,
  BackwardWeights/Im2colGemm} at N=256, bf16, through
  ``primkit_conv_run_device`` exactly as bench.py issues them — so the kernel
  template instances checked here are the ones the bench times. The
  instance string (``primkit_handle_last_variant``) is recorded per problem
  (PK_VARIANT_LOG=<path> writes the table) and must name a tensor-core kernel.
* cfg1: fp32 3x3 N=8 C=K=64 56x56 Direct, full tensor vs the oracle.
* cfg2: fused conv+bias+ReLU plans at N=64 (1x1 64->256 and 3x3 64->64),
  fp32 and bf16, fused and unfused, vs the oracle epilogue formula.
* cfg3: VGG-16's 13 layers at N=128, bf16, ImplicitGemm and Winograd.
* cfg4: conv + training BN (+ReLU) fused forward for all 53 ResNet-50 layers
  at N=256: batch statistics vs the reference formula on the stored conv
  output, running-stat update, normalised output.

Full-size outputs are checked on >= 4096 sampled coordinates against the
oracle's f64 direct formula on the same device-layout operands
(oracle.sample_*); tolerances as north_star states: bf16
<= 1e-2 relative L2 vs the fp32/f64 oracle, fp32 <= 1e-4 (Winograd 1e-3).
Reference: proj/tests/acceptance.cpp:86-152 (random conv vs the f64 oracle).
"""
import ctypes as C
import json
import os
import zlib

import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import problem
from paper_1910_00078_b200.resnet50 import resnet50_layers, vgg16_layers

from conftest import max_rel, rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

NS = 4096          # sampled output coordinates per forward / backward-data problem
WG_K, WG_T = 64, 64  # backward weights: 64 output channels x 64 (r, s, c) taps
_VARIANTS = {}


def pitch(c):
    return (c + 7) // 8 * 8


class Dev:
    """A stream-bound primkit handle plus torch device buffers (the bench's setup)."""

    def __init__(self, lib):
        self.L = lib
        self.stream = torch.cuda.current_stream()
        self.h = C.c_void_p()
        lib.check(lib.lib.primkit_handle_create_with_stream(C.c_void_p(self.stream.cuda_stream), 0,
                                                            C.byref(self.h)))
        self.gen = torch.Generator(device="cuda")

    def rand(self, shape, c_real=None, seed=0, dtype=torch.bfloat16):
        self.gen.manual_seed(seed)
        t = (torch.rand(shape, generator=self.gen, device="cuda", dtype=torch.float32) * 2 - 1).to(dtype)
        if c_real is not None and c_real != shape[-1]:
            t[..., c_real:] = 0
        return t

    def workspace(self, p, solver):
        ws = C.c_uint64()
        self.L.check(self.L.lib.primkit_conv_device_workspace(self.h, C.byref(p), solver.encode(),
                                                              C.byref(ws)))
        return torch.empty(max(int(ws.value), 256), dtype=torch.uint8, device="cuda")

    def run(self, p, solver, a, b, out):
        ws = self.workspace(p, solver)
        self.L.check(self.L.lib.primkit_conv_run_device(
            self.h, C.byref(p), solver.encode(), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
            C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel())))
        kname, var = C.create_string_buffer(128), C.create_string_buffer(1024)
        self.L.check(self.L.lib.primkit_handle_last_kernel(self.h, kname, 128))
        self.L.check(self.L.lib.primkit_handle_last_variant(self.h, var, 1024))
        torch.cuda.synchronize()
        return kname.value.decode(), var.value.decode()


@pytest.fixture(scope="module")
def dev(lib):
    d = Dev(lib)
    yield d
    d.L.lib.primkit_handle_destroy(d.h)
    log = os.environ.get("PK_VARIANT_LOG")
    if log and _VARIANTS:
        with open(log, "w") as f:
            json.dump(_VARIANTS, f, indent=1, sort_keys=True)


def host(t):
    """Device tensor -> host array in the same layout (bf16 as raw uint16)."""
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def as_f64(a):
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def sample_idx(rng, n0, n1, n2, n3, ns=NS):
    """ns coordinates (a, b, c, d) incl. both corners."""
    idx = np.stack([rng.integers(0, m, ns) for m in (n0, n1, n2, n3)], 1)
    idx[0] = (0, 0, 0, 0)
    idx[1] = (n0 - 1, n1 - 1, n2 - 1, n3 - 1)
    return idx


def check_samples(got, want, tol, what):
    err = rel_l2(got, want)
    assert err <= tol, f"{what}: rel-L2 {err:.3e} > {tol} (max-rel {max_rel(got, want):.3e})"
    return err


def layer_problem(L, n, direction, etype=abi.BF16):
    return problem(n=n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad, stride=L.stride,
                   direction=direction, etype=etype)


# ---- bench step: 53 layers x 3 directions at N=256 --------------------------

STEP = [("ImplicitGemm", abi.FORWARD), ("Im2colGemm", abi.BACKWARD_DATA),
        ("Im2colGemm", abi.BACKWARD_WEIGHTS)]


@pytest.mark.parametrize("L", resnet50_layers(), ids=lambda L: L.name)
def test_resnet50_step_layer_n256(lib, dev, L):
    n = 256
    rng = np.random.default_rng(zlib.crc32(L.name.encode()))
    ho = L.out_h
    cp, kp = pitch(L.c), pitch(L.k)
    x = dev.rand((n, L.h, L.h, cp), L.c, seed=1)
    w = dev.rand((L.k, L.r, L.r, cp), L.c, seed=2)
    dy = dev.rand((n, ho, ho, kp), L.k, seed=3)
    y = torch.empty((n, ho, ho, kp), dtype=torch.bfloat16, device="cuda")
    dx = torch.empty_like(x)
    dw = torch.empty_like(w)
    xh, wh, dyh = host(x), host(w), host(dy)
    for solver, d in STEP:
        p = layer_problem(L, n, d)
        a, b, out = {abi.FORWARD: (x, w, y), abi.BACKWARD_DATA: (dy, w, dx),
                     abi.BACKWARD_WEIGHTS: (dy, x, dw)}[d]
        kern, var = dev.run(p, solver, a, b, out)
        _VARIANTS[f"{L.name}/{['fwd', 'bwd_data', 'bwd_weights'][d]}"] = {"kernel": kern, "variant": var}
        assert kern.startswith(("igemm_tc", "stem_fused")), kern
        assert var, f"{L.name} dir {d}: no tensor-core kernel instance recorded ({kern})"
        oh = host(out)
        if d == abi.FORWARD:
            idx = sample_idx(rng, n, L.k, ho, ho)
            want = oracle.sample_forward(p, xh, wh, idx)
            got = as_f64(oh[idx[:, 0], idx[:, 2], idx[:, 3], idx[:, 1]])
            if kp != L.k:
                assert not oh[..., L.k:].any(), "forward pad lanes must stay zero"
        elif d == abi.BACKWARD_DATA:
            idx = sample_idx(rng, n, L.c, L.h, L.h)
            want = oracle.sample_backward_data(p, dyh, wh, idx)
            got = as_f64(oh[idx[:, 0], idx[:, 2], idx[:, 3], idx[:, 1]])
            if cp != L.c:
                assert not oh[..., L.c:].any(), "dX pad lanes must stay zero"
        else:
            ks = rng.choice(L.k, min(WG_K, L.k), replace=False)
            ks[0] = 0
            taps = np.stack([rng.integers(0, L.r, WG_T), rng.integers(0, L.r, WG_T),
                             rng.integers(0, L.c, WG_T)], 1)
            want = oracle.sample_backward_weights(p, dyh, xh, ks, taps).ravel()
            got = as_f64(oh[ks[:, None], taps[None, :, 0], taps[None, :, 1], taps[None, :, 2]]).ravel()
        check_samples(got, want, 1e-2, f"{L.name} dir {d} {var}")


# ---- cfg1: fp32 3x3 Direct, full tensor ---------------------------------------

def test_cfg1_direct_fp32_full_tensor(lib):
    rng = np.random.default_rng(101)
    p = problem(n=8, c=64, h=56, w=56, k=64, y=3, x=3, pad=1)
    x = rng.uniform(-1, 1, (8, 64, 56, 56)).astype(np.float32)
    w = rng.uniform(-1, 1, (64, 64, 3, 3)).astype(np.float32)
    h = lib.handle()
    got = h.conv_run(p, "Direct", x, w)
    # fp32 on the tensor cores at fp32 accuracy (3xTF32); PK_TF32X3=0 selects direct_simt
    assert h.last_kernel() in ("tf32x3_tc_fwd", "direct_simt"), h.last_kernel()
    want = oracle.conv_forward(p, x, w)
    assert rel_l2(got, want) <= 1e-4
    assert max_rel(got, want) <= 1e-4


# ---- cfg2: fused conv+bias+ReLU at N=64 ---------------------------------------

def _to_dev(a, pit):
    n, c, hh, ww = a.shape
    out = np.zeros((n, hh, ww, pit), np.float32)
    out[..., :c] = a.transpose(0, 2, 3, 1)
    return out


CFG2 = [
    # (name, C, K, f, pad, etype, algo label, ops)
    ("1x1_f32_cba", 64, 256, 1, 0, abi.F32, "Direct", "cba"),
    ("1x1_bf16_cba", 64, 256, 1, 0, abi.BF16, "Direct", "cba"),
    ("3x3_f32_cba_winograd", 64, 64, 3, 1, abi.F32, "Winograd", "cba"),
    ("3x3_bf16_cbna", 64, 64, 3, 1, abi.BF16, "Direct", "cbna"),
]


@pytest.mark.parametrize("cfg", CFG2, ids=lambda c: c[0])
@pytest.mark.parametrize("unfused", [0, 1])
def test_cfg2_fusion_n64(lib, cfg, unfused):
    name, c, k, f, pad, et, algo, ops = cfg
    n, hw = 64, 56
    rng = np.random.default_rng(202)
    bf = et == abi.BF16
    q = oracle.round_bf16 if bf else (lambda a: a)
    x = q(rng.uniform(-1, 1, (n, c, hw, hw)).astype(np.float32))
    w = q(rng.uniform(-1, 1, (k, c, f, f)).astype(np.float32))
    bias = rng.uniform(-1, 1, k).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, k).astype(np.float32)
    beta = rng.uniform(-1, 1, k).astype(np.float32)
    mean = rng.uniform(-1, 1, k).astype(np.float32)
    var = (1 + np.abs(rng.uniform(-1, 1, k))).astype(np.float32)
    h = lib.handle()
    plan = lib.fusion_plan((n, c, hw, hw), et)
    lib.check(plan.add_conv((k, c, f, f), pad=pad, algo=algo))
    lib.check(plan.add_bias(k))
    if ops == "cbna":
        lib.check(plan.add_batchnorm(abi.BN_SPATIAL))
    lib.check(plan.add_activation(abi.RELU))
    lib.check(plan.compile(h))
    plan.set_args(filter=w, bias=bias, gamma=gamma, beta=beta, mean=mean, var=var, eps=1e-5)
    out = plan.execute(h, x, unfused=bool(unfused))
    p = problem(n=n, c=c, h=hw, w=hw, k=k, y=f, x=f, pad=pad)
    idx = sample_idx(rng, n, k, hw, hw)
    acc = oracle.sample_forward(p, np.ascontiguousarray(_to_dev(x, pitch(c))),
                                np.ascontiguousarray(_to_dev(w, pitch(c))), idx, bf16=False)
    kk = idx[:, 1]
    want = acc + bias[kk]
    if ops == "cbna":
        want = (want - mean[kk]) / np.sqrt(var[kk].astype(np.float64) + 1e-5) * gamma[kk] + beta[kk]
    want = np.maximum(want, 0)
    got = out[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]]
    tol = 1e-2 if bf else (1e-3 if algo == "Winograd" else 1e-4)
    check_samples(got, want, tol, name)


# ---- cfg3: VGG-16 at N=128, ImplicitGemm and Winograd -----------------------------

@pytest.mark.parametrize("solver", ["ImplicitGemm", "Winograd"])
@pytest.mark.parametrize("L", vgg16_layers(), ids=lambda L: L.name)
def test_cfg3_vgg16_n128(lib, dev, L, solver):
    n = 128
    rng = np.random.default_rng(303)
    cp, kp = pitch(L.c), pitch(L.k)
    x = dev.rand((n, L.h, L.h, cp), L.c, seed=11)
    w = dev.rand((L.k, L.r, L.r, cp), L.c, seed=12)
    y = torch.empty((n, L.out_h, L.out_h, kp), dtype=torch.bfloat16, device="cuda")
    p = layer_problem(L, n, abi.FORWARD)
    kern, var = dev.run(p, solver, x, w, y)
    _VARIANTS[f"{L.name}/fwd/{solver}"] = {"kernel": kern, "variant": var}
    idx = sample_idx(rng, n, L.k, L.out_h, L.out_h)
    want = oracle.sample_forward(p, host(x), host(w), idx)
    yh = host(y)
    got = as_f64(yh[idx[:, 0], idx[:, 2], idx[:, 3], idx[:, 1]])
    check_samples(got, want, 1e-2, f"{L.name} {solver} {kern}")


# ---- cfg4: conv + training BN (+ReLU) fused forward at N=256 ----------------------

@pytest.mark.parametrize("L", resnet50_layers(), ids=lambda L: L.name)
def test_cfg4_conv_bn_train_n256(lib, dev, L):
    n, eps, mom = 256, 1e-5, 0.1
    rng = np.random.default_rng(404)
    cp, kp, ho = pitch(L.c), pitch(L.k), L.out_h
    x = dev.rand((n, L.h, L.h, cp), L.c, seed=21)
    w = dev.rand((L.k, L.r, L.r, cp), L.c, seed=22)
    conv_out = torch.empty((n, ho, ho, kp), dtype=torch.bfloat16, device="cuda")
    y = torch.empty_like(conv_out)
    f32 = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda")  # noqa: E731
    gamma_h = rng.uniform(0.5, 1.5, L.k).astype(np.float32)
    beta_h = rng.uniform(-1, 1, L.k).astype(np.float32)
    rm_h = rng.uniform(-1, 1, L.k).astype(np.float32)
    rv_h = (1 + np.abs(rng.uniform(-1, 1, L.k))).astype(np.float32)
    gamma, beta, rm, rv = f32(gamma_h), f32(beta_h), f32(rm_h), f32(rv_h)
    sm, si = torch.empty(L.k, device="cuda"), torch.empty(L.k, device="cuda")
    p = layer_problem(L, n, abi.FORWARD)
    ws = C.c_uint64()
    lib.check(lib.lib.primkit_conv_bn_workspace(dev.h, C.byref(p), b"ImplicitGemm", C.byref(ws)))
    wsb = torch.empty(int(ws.value), dtype=torch.uint8, device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    lib.check(lib.lib.primkit_conv_bn_forward_train_device(
        dev.h, C.byref(p), b"ImplicitGemm", P(x), P(w), P(gamma), P(beta), P(rm), P(rv),
        C.c_float(eps), C.c_float(mom), P(conv_out), P(y), P(sm), P(si), 1, P(wsb),
        C.c_size_t(wsb.numel())))
    torch.cuda.synchronize()
    co = host(conv_out)
    # the stored convolution output itself
    idx = sample_idx(rng, n, L.k, ho, ho)
    want = oracle.sample_forward(p, host(x), host(w), idx)
    check_samples(as_f64(co[idx[:, 0], idx[:, 2], idx[:, 3], idx[:, 1]]), want, 1e-2, L.name + " conv")
    # batch statistics of exactly the stored values (reference formula, double sums)
    mean_r, inv_r, var_r = oracle.bn_stats_device(co[..., :L.k] if kp != L.k else co, L.k, eps)
    np.testing.assert_allclose(sm.cpu().numpy(), mean_r, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(si.cpu().numpy(), inv_r, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(rm.cpu().numpy(), (1 - mom) * rm_h + mom * mean_r, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(rv.cpu().numpy(), (1 - mom) * rv_h + mom * var_r, rtol=1e-5, atol=1e-6)
    # normalised + ReLU output on the sampled coordinates
    kk = idx[:, 1]
    cv = as_f64(co[idx[:, 0], idx[:, 2], idx[:, 3], kk])
    want_y = np.maximum(gamma_h[kk] * (cv - mean_r[kk]) * inv_r[kk] + beta_h[kk], 0)
    got_y = as_f64(host(y)[idx[:, 0], idx[:, 2], idx[:, 3], kk])
    check_samples(got_y, want_y, 1e-2, L.name + " bn")
