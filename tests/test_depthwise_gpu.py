"""Depthwise convolution (groups == C == K) parity on the GPU through the C ABI.

Direct and ImplicitGemm route these problems to the channel-vector depthwise
kernels (depthwise.cu); every direction, f32 and bf16, against the oracle's
grouped direct convolution (reference proj/src/core/conv.cpp:99-133, 716-756,
816-850 with cg == kg == 1). Tolerances as in test_conv_gpu.py: f32 <= 1e-4,
bf16 <= 1e-2 relative L2."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu

SHAPES = [
    dict(n=2, c=16, h=9, w=9, k=16, y=3, x=3, pad=1, groups=16),
    dict(n=1, c=24, h=13, w=11, k=24, y=5, x=5, pad=2, stride=2, groups=24),      # 8-channel blocks
    dict(n=2, c=64, h=10, w=10, k=64, y=3, x=3, pad=2, dilation=2, groups=64),
    dict(n=3, c=5, h=8, w=7, k=5, y=3, x=3, pad=1, stride=2, groups=5),           # pad lanes
    dict(n=1, c=96, h=12, w=12, k=96, y=7, x=7, pad=3, groups=96),                # 49 taps
    dict(n=2, c=32, h=9, w=8, k=32, y=3, x=2, pad_h=0, pad_w=1, groups=32),       # ragged
    dict(n=4, c=96, h=28, w=28, k=96, y=3, x=3, pad=1, groups=96),                # many chunks
    dict(n=2, c=40, h=7, w=10, k=40, y=3, x=3, pad_h=0, pad_w=2, groups=40),      # 3x3 s1 quads, ragged
    dict(n=1, c=8, h=5, w=3, k=8, y=3, x=3, pad=1, groups=8),                     # row shorter than a quad
]


def _cases():
    for i in range(len(SHAPES)):
        for et in (abi.F32, abi.BF16):
            for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
                yield pytest.param(i, et, d, id=f"dw{i}-{'bf16' if et else 'f32'}-d{d}")


def _run(lib, p, rng, bf16):
    sa, sb, _ = operand_shapes(lib, p)
    a = rng.uniform(-1, 1, sa).astype(np.float32)
    b = rng.uniform(-1, 1, sb).astype(np.float32)
    if bf16:
        a, b = oracle.round_bf16(a), oracle.round_bf16(b)
    if p.direction == abi.FORWARD:
        want = oracle.conv_forward(p, a, b)
    elif p.direction == abi.BACKWARD_DATA:
        want = oracle.conv_backward_data(p, a, b)
    else:
        want = oracle.conv_backward_weights(p, a, b)
    return a, b, want


@pytest.mark.parametrize("si,et,direction", list(_cases()))
def test_depthwise_parity(lib, si, et, direction):
    rng = np.random.default_rng(700 + si)
    p = problem(**SHAPES[si], direction=direction, etype=et)
    h = lib.handle()
    a, b, want = _run(lib, p, rng, et == abi.BF16)
    ran = 0
    for s in ("Direct", "ImplicitGemm", "Im2colGemm"):
        if not h.is_applicable(s, p):
            continue
        got = h.conv_run(p, s, a, b)
        assert h.last_kernel().startswith("depthwise"), h.last_kernel()
        tol = 1e-2 if et == abi.BF16 else 1e-4
        err = rel_l2(got, want)
        assert err <= tol, f"{s} {h.last_kernel()} rel-L2 {err:.3e}"
        if et == abi.BF16:
            assert np.array_equal(oracle.round_bf16(got), got)
        again = h.conv_run(p, s, a, b)
        assert np.array_equal(got, again), "depthwise result is not deterministic"
        ran += 1
    assert ran >= 1


GROUPED = [
    dict(n=2, c=32, h=9, w=9, k=64, y=3, x=3, pad=1, groups=4),                  # cg 8, kg 16
    dict(n=1, c=32, h=11, w=10, k=128, y=5, x=5, pad=2, stride=2, groups=2),     # cg 16, kg 64, 25 taps
    dict(n=2, c=256, h=8, w=8, k=64, y=3, x=3, pad=2, dilation=2, groups=8),     # cg 32, kg 8
    dict(n=4, c=256, h=14, w=14, k=256, y=3, x=3, pad=1, groups=32),             # ResNeXt-like
    dict(n=1, c=64, h=6, w=7, k=64, y=1, x=1, groups=8),                         # 1x1
]


GROUPED_KERNEL = {abi.FORWARD: "grouped_simt", abi.BACKWARD_DATA: "grouped_simt_bwd_data",
                  abi.BACKWARD_WEIGHTS: "grouped_simt_bwd_weights"}


@pytest.mark.parametrize("si", range(len(GROUPED)))
@pytest.mark.parametrize("et", [abi.F32, abi.BF16])
@pytest.mark.parametrize("direction", [abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS])
def test_grouped_parity(lib, si, et, direction):
    rng = np.random.default_rng(800 + si)
    p = problem(**GROUPED[si], direction=direction, etype=et)
    h = lib.handle()
    a, b, want = _run(lib, p, rng, et == abi.BF16)
    ran = 0
    for s in ("Direct", "ImplicitGemm", "Im2colGemm"):
        if not h.is_applicable(s, p):
            continue
        got = h.conv_run(p, s, a, b)
        sh = GROUPED[si]
        cg, kg = sh["c"] // sh["groups"], sh["k"] // sh["groups"]
        staged = sh["y"] * sh["x"] * max(cg, kg) * 64 * 4  # filter slice in smem (fwd / bwd-data)
        if direction == abi.BACKWARD_WEIGHTS or staged <= 160 * 1024:
            assert h.last_kernel() == GROUPED_KERNEL[direction], h.last_kernel()
        tol = 1e-2 if et == abi.BF16 else 1e-4
        err = rel_l2(got, want)
        assert err <= tol, f"{s} {h.last_kernel()} rel-L2 {err:.3e}"
        assert np.array_equal(got, h.conv_run(p, s, a, b)), "not deterministic"
        ran += 1
    assert ran >= 1
