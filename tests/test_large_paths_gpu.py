"""Full-size paths that only engage at ResNet-50 scale (grids of >= 74 SM
pairs, whole-image halo k-blocks), checked against a second GPU algorithm —
the fp32 SIMT Direct kernel on the same bf16-rounded inputs — plus sampled
output coordinates against the CPU oracle formula:

* CTA-pair (cta_group::2) plain GEMM, forward with a fused bias+ReLU epilogue
  through the fusion-plan API, and backward data;
* CTA-pair TMA rectangle convolution (256-wide tiles, stride 2);
* padded-grid halo wgrad with ragged image rows and fewer k-blocks than SMs.

Tolerance: bf16 outputs within 1e-2 relative L2 of the fp32 reference."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _rand(rng, shape):
    return oracle.round_bf16(rng.uniform(-1, 1, shape).astype(np.float32))


def _check_against_direct(h, p, a, b, solver, kernel_prefix):
    got = h.conv_run(p, solver, a, b)
    kern = h.last_kernel()
    assert kern.startswith(kernel_prefix), kern
    pf = problem(n=p.n, c=p.c, h=p.h, w=p.w, k=p.k, y=p.y, x=p.x, pad_h=p.pad_h, pad_w=p.pad_w,
                 stride_h=p.stride_h, stride_w=p.stride_w, direction=p.direction, etype=abi.F32)
    ref = h.conv_run(pf, "Direct", a, b)  # fp32 SIMT on the same (bf16-valued) inputs
    err = rel_l2(got, ref)
    assert err <= 1e-2, (kern, err)
    return got


def test_pair_gemm_forward_fused_bias_relu(lib):
    rng = np.random.default_rng(71)
    n, c, hw, k = 8, 512, 56, 256
    x, w = _rand(rng, (n, c, hw, hw)), _rand(rng, (k, c, 1, 1))
    bias = rng.uniform(-1, 1, k).astype(np.float32)
    h = lib.handle()
    plan = lib.fusion_plan((n, c, hw, hw), abi.BF16)
    lib.check(plan.add_conv((k, c, 1, 1)))
    lib.check(plan.add_bias(k))
    lib.check(plan.add_activation(abi.RELU))
    lib.check(plan.compile(h))
    plan.set_args(filter=w, bias=bias)
    out = plan.execute(h, x)
    # reference: fp32 Direct conv on the GPU + bias + ReLU
    p = problem(n=n, c=c, h=hw, w=hw, k=k)
    ref = np.maximum(h.conv_run(p, "Direct", x, w) + bias[None, :, None, None], 0)
    assert rel_l2(out, ref) <= 1e-2
    # sampled coordinates against the CPU formula
    for (i, kk, yy, xx) in [(0, 0, 0, 0), (7, 255, 55, 55), (3, 100, 20, 31)]:
        v = max(float(np.dot(x[i, :, yy, xx].astype(np.float64), w[kk, :, 0, 0])) + bias[kk], 0.0)
        assert abs(out[i, kk, yy, xx] - v) <= 2e-2 * (1 + abs(v))


def test_pair_gemm_backward_data(lib):
    rng = np.random.default_rng(72)
    p = problem(n=8, c=256, h=56, w=56, k=512, direction=abi.BACKWARD_DATA, etype=abi.BF16)
    sa, sb, _ = operand_shapes(lib, p)
    h = lib.handle()
    _check_against_direct(h, p, _rand(rng, sa), _rand(rng, sb), "Im2colGemm", "igemm_tc_dgrad")


def test_pair_rectangle_stride2_forward(lib):
    rng = np.random.default_rng(73)
    p = problem(n=128, c=256, h=28, w=28, k=256, y=3, x=3, pad=1, stride=2, etype=abi.BF16)
    sa, sb, _ = operand_shapes(lib, p)
    h = lib.handle()
    _check_against_direct(h, p, _rand(rng, sa), _rand(rng, sb), "ImplicitGemm", "igemm_tc_fwd")


@pytest.mark.parametrize("shape", [dict(n=1, h=57, w=57), dict(n=3, h=30, w=22)])
def test_halo_wgrad_ragged(lib, shape):
    rng = np.random.default_rng(74)
    p = problem(c=64, k=64, y=3, x=3, pad=1, direction=abi.BACKWARD_WEIGHTS, etype=abi.BF16, **shape)
    sa, sb, _ = operand_shapes(lib, p)
    dy, x = _rand(rng, sa), _rand(rng, sb)
    h = lib.handle()
    got = h.conv_run(p, "Im2colGemm", dy, x)
    want = oracle.conv_backward_weights(p, dy, x)
    assert rel_l2(got, want) <= 1e-2
