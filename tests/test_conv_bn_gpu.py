"""Convolution + training batch-norm (+ReLU) with the BN statistics computed
in the convolution epilogue (BASELINE cfg4, primkit_conv_bn_forward_train_device)
against the oracle: conv output within the bf16 tolerance of the fp32 oracle
convolution, and the batch statistics / normalised output / running statistics
against the reference BN (primitives.cpp:61-96) evaluated on the very conv
output the kernel stored (isolates the fused statistics from conv rounding).
Also: fused == unfused (conv, then standalone BN) on the same device tensors."""
import ctypes as C

import os

import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SHAPES = [
    dict(n=4, c=64, h=14, w=14, k=256, y=1, x=1),                  # PLAIN 1x1 (conv_tc)
    dict(n=2, c=64, h=28, w=28, k=64, y=3, x=3, pad=1),            # TMA rectangles
    dict(n=2, c=128, h=15, w=15, k=128, y=3, x=3, pad=1, stride=2),  # strided, ragged
    dict(n=2, c=3, h=64, w=64, k=64, y=7, x=7, pad=3, stride=2),   # fused stem
    dict(n=3, c=256, h=9, w=9, k=320, y=1, x=1),                   # K not a multiple of 64
]


def _nhwc(a, pitch):
    """NCHW float32 numpy -> NHWC bf16 device tensor with zero pad lanes."""
    t = torch.from_numpy(np.ascontiguousarray(a)).permute(0, 2, 3, 1).contiguous()
    out = torch.zeros(t.shape[:-1] + (pitch,), dtype=torch.bfloat16)
    out[..., : t.shape[-1]] = t.to(torch.bfloat16)
    return out.cuda()


def _nchw(t, c):
    return t[..., :c].float().permute(0, 3, 1, 2).contiguous().cpu().numpy()


def _vp(t):
    return C.c_void_p(t.data_ptr())


def _run(lib, h, p, x, w, gamma, beta, rm, rv, relu, fused=True):
    k = p.k
    ho = (p.h + 2 * p.pad_h - p.y) // p.stride_h + 1
    wo = (p.w + 2 * p.pad_w - p.x) // p.stride_w + 1
    kp = lib.channel_pitch(k)
    conv_out = torch.zeros((p.n, ho, wo, kp), dtype=torch.bfloat16, device="cuda")
    y = torch.zeros_like(conv_out)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    g, b, rmd, rvd = dev(gamma), dev(beta), dev(rm), dev(rv)
    sm, si = torch.zeros(k, device="cuda"), torch.zeros(k, device="cuda")
    if fused:
        ws = C.c_uint64()
        lib.check(lib.lib.primkit_conv_bn_workspace(h.ptr, C.byref(p), b"ImplicitGemm", C.byref(ws)))
        wsb = torch.empty(max(ws.value, 256), dtype=torch.uint8, device="cuda")
        lib.check(lib.lib.primkit_conv_bn_forward_train_device(
            h.ptr, C.byref(p), b"ImplicitGemm", _vp(x), _vp(w), _vp(g), _vp(b), _vp(rmd), _vp(rvd),
            C.c_float(1e-5), C.c_float(0.1), _vp(conv_out), _vp(y), _vp(sm), _vp(si), int(relu),
            _vp(wsb), C.c_size_t(wsb.numel())))
    else:
        ws = C.c_uint64()
        lib.check(lib.lib.primkit_conv_device_workspace(h.ptr, C.byref(p), b"ImplicitGemm",
                                                        C.byref(ws)))
        wsb = torch.empty(max(ws.value, 256), dtype=torch.uint8, device="cuda")
        lib.check(lib.lib.primkit_conv_run_device(h.ptr, C.byref(p), b"ImplicitGemm", _vp(x), _vp(w),
                                                  _vp(conv_out), _vp(wsb), C.c_size_t(wsb.numel())))
        dims = (C.c_int64 * 4)(p.n, k, ho, wo)
        lib.check(lib.lib.primkit_batchnorm_forward_train_device(
            h.ptr, dims, abi.BF16, _vp(conv_out), _vp(g), _vp(b), _vp(rmd), _vp(rvd),
            C.c_float(1e-5), C.c_float(0.1), _vp(y), _vp(sm), _vp(si), int(relu)))
    torch.cuda.synchronize()
    return (_nchw(conv_out, k), _nchw(y, k), sm.cpu().numpy(), si.cpu().numpy(),
            rmd.cpu().numpy(), rvd.cpu().numpy())


@pytest.mark.parametrize("si", range(len(SHAPES)))
@pytest.mark.parametrize("relu", [0, 1])
def test_conv_bn_forward_train(lib, si, relu):
    rng = np.random.default_rng(500 + si)
    s = SHAPES[si]
    p = problem(**s, etype=abi.BF16)
    xn = oracle.round_bf16(rng.uniform(-1, 1, (p.n, p.c, p.h, p.w)).astype(np.float32))
    wn = oracle.round_bf16(rng.uniform(-1, 1, (p.k, p.c, p.y, p.x)).astype(np.float32))
    cp = lib.channel_pitch(p.c)
    x = _nhwc(xn, cp)
    w = _nhwc(wn, cp)  # [K][R][S][pitch]
    gamma = rng.uniform(0.5, 1.5, p.k).astype(np.float32)
    beta = rng.uniform(-1, 1, p.k).astype(np.float32)
    rm = rng.uniform(-1, 1, p.k).astype(np.float32)
    rv = (1 + np.abs(rng.uniform(-1, 1, p.k))).astype(np.float32)
    h = lib.handle()
    os.environ["PK_CBN_FUSE"] = "1"  # always the epilogue-statistics path here
    try:
        conv, y, sm, sinv, rm_out, rv_out = _run(lib, h, p, x, w, gamma, beta, rm, rv, relu)
    finally:
        os.environ.pop("PK_CBN_FUSE", None)
    assert "bn_stats_epilogue" in h.last_kernel(), h.last_kernel()
    # the convolution itself: bf16 tolerance vs the fp32 oracle
    assert rel_l2(conv, oracle.conv_forward(p, xn, wn)) <= 1e-2
    # BN semantics on the stored conv output (reference, double accumulation)
    want_y, want_m, want_i, want_rm, want_rv = oracle.bn_forward_train(
        abi.BN_SPATIAL, conv, gamma, beta, rm.copy(), rv.copy(), 1e-5, 0.1, bf16=True)
    np.testing.assert_allclose(sm, want_m, rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(sinv, want_i, rtol=1e-4)
    np.testing.assert_allclose(rm_out, want_rm, rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(rv_out, want_rv, rtol=1e-4, atol=1e-5)
    if relu:
        want_y = np.maximum(want_y, 0)
    assert rel_l2(y, want_y) <= 1e-2
    # fused == unfused (conv kernel, then the standalone BN kernels)
    _, y2, sm2, si2, _, _ = _run(lib, h, p, x, w, gamma, beta, rm, rv, relu, fused=False)
    np.testing.assert_allclose(sm, sm2, rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(sinv, si2, rtol=1e-4)
    assert rel_l2(y, y2) <= 1e-2


BWD_SHAPES = [  # the BackwardData convolution of the NEXT layer; its dX feeds the BN
    dict(n=4, c=64, h=14, w=14, k=256, y=1, x=1),                  # PLAIN 1x1 dgrad
    dict(n=2, c=64, h=28, w=28, k=64, y=3, x=3, pad=1),            # TMA dgrad
    dict(n=2, c=128, h=15, w=15, k=128, y=3, x=3, pad=1, stride=2),  # phased dgrad
    dict(n=2, c=256, h=14, w=14, k=512, y=1, x=1, stride=2),       # phased 1x1
]


@pytest.mark.parametrize("si", range(len(BWD_SHAPES)))
@pytest.mark.parametrize("relu", [0, 1])
def test_dgrad_bn_backward(lib, si, relu, monkeypatch):
    rng = np.random.default_rng(700 + si)
    p = problem(**BWD_SHAPES[si], direction=abi.BACKWARD_DATA, etype=abi.BF16)
    ho = (p.h + 2 * p.pad_h - p.y) // p.stride_h + 1
    wo = (p.w + 2 * p.pad_w - p.x) // p.stride_w + 1
    cp, kp = lib.channel_pitch(p.c), lib.channel_pitch(p.k)
    dyn = oracle.round_bf16(rng.uniform(-1, 1, (p.n, p.k, ho, wo)).astype(np.float32))
    wn = oracle.round_bf16(rng.uniform(-1, 1, (p.k, p.c, p.y, p.x)).astype(np.float32))
    bxn = oracle.round_bf16(rng.uniform(-2, 2, (p.n, p.c, p.h, p.w)).astype(np.float32))
    gamma = rng.uniform(0.5, 1.5, p.c).astype(np.float32)
    beta = rng.uniform(-0.5, 0.5, p.c).astype(np.float32)
    _, smean, sinv, _, _ = oracle.bn_forward_train(abi.BN_SPATIAL, bxn, gamma, beta,
                                                   np.zeros(p.c, np.float32),
                                                   np.ones(p.c, np.float32), 1e-5, 0.1, bf16=True)
    dy, w, bx = _nhwc(dyn, kp), _nhwc(wn, cp), _nhwc(bxn, cp)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    g, b, sm, si_ = dev(gamma), dev(beta), dev(smean), dev(sinv)
    h = lib.handle()
    out = []
    # fold: dgrad + one-launch BN backward, mask from the BN input (default);
    # epi: statistics in the dgrad epilogue (PK_CBN_BWD_EPI=1); Direct: unfused
    for mode in ("fold", "epi", "unfused"):
        fused = mode != "unfused"
        monkeypatch.setenv("PK_CBN_BWD_EPI", "1" if mode == "epi" else "0")
        dz = torch.zeros((p.n, p.h, p.w, cp), dtype=torch.bfloat16, device="cuda")
        bdx = torch.zeros_like(dz)
        dg, db = torch.zeros(p.c, device="cuda"), torch.zeros(p.c, device="cuda")
        ws = C.c_uint64()
        lib.check(lib.lib.primkit_conv_bn_workspace(h.ptr, C.byref(p), b"Im2colGemm", C.byref(ws)))
        wsb = torch.empty(max(ws.value, 256), dtype=torch.uint8, device="cuda")
        solver = b"Im2colGemm" if fused else b"Direct"  # Direct: unfused fallback path
        if not fused:
            lib.check(lib.lib.primkit_conv_bn_workspace(h.ptr, C.byref(p), solver, C.byref(ws)))
            wsb = torch.empty(max(ws.value, 256), dtype=torch.uint8, device="cuda")
        lib.check(lib.lib.primkit_conv_backward_data_bn_device(
            h.ptr, C.byref(p), solver, _vp(dy), _vp(w), _vp(dz), _vp(bx), _vp(g), _vp(b), _vp(sm),
            _vp(si_), int(relu), _vp(bdx), _vp(dg), _vp(db), _vp(wsb), C.c_size_t(wsb.numel())))
        torch.cuda.synchronize()
        if mode == "epi":
            assert "bn_bwd_stats_epilogue" in h.last_kernel(), h.last_kernel()
        if mode == "fold":
            assert "bn_bwd_fold" in h.last_kernel(), h.last_kernel()
        out.append((_nchw(dz, p.c), _nchw(bdx, p.c), dg.cpu().numpy(), db.cpu().numpy()))
    (dz_f, bdx_f, dg_f, db_f), (dz_e, bdx_e, dg_e, db_e), (dz_u, bdx_u, dg_u, db_u) = out
    assert rel_l2(bdx_e, bdx_f) <= 2e-2 and rel_l2(dg_e, dg_f) <= 2e-2
    assert rel_l2(dz_f, oracle.conv_backward_data(p, dyn, wn)) <= 1e-2
    # reference BN backward on the stored dz, ReLU mask of the forward output
    mask = 1.0
    if relu:
        fwd = gamma[None, :, None, None] * (bxn - smean[None, :, None, None]) * \
            sinv[None, :, None, None] + beta[None, :, None, None]
        mask = (fwd > 0).astype(np.float32)
    want_dx, want_dg, want_db = oracle.bn_backward(abi.BN_SPATIAL, bxn, dz_f * mask, gamma, smean,
                                                   sinv, bf16=True)
    np.testing.assert_allclose(db_f, want_db, rtol=2e-2, atol=2e-2)
    np.testing.assert_allclose(dg_f, want_dg, rtol=2e-2, atol=2e-2)
    assert rel_l2(bdx_f, want_dx) <= 1e-2
    # fused == unfused composition (Direct dgrad + standalone BN backward)
    assert rel_l2(dz_f, dz_u) <= 1e-2
    assert rel_l2(bdx_f, bdx_u) <= 2e-2
