"""Full-size paths that only engage at ResNet-50 scale (grids of >= 74 SM
pairs, whole-image halo k-blocks), checked against the CPU oracle's f64
direct formula on 4096 sampled output coordinates (oracle.sample_*):

* CTA-pair (cta_group::2) plain GEMM, forward with a fused bias+ReLU epilogue
  through the fusion-plan API, and backward data;
* CTA-pair TMA rectangle convolution (256-wide tiles, stride 2);
* CTA-pair TMA rectangle backward data (conv4_x / conv5_x 3x3, >= 74 pair tiles);
* padded-grid halo wgrad with ragged image rows and fewer k-blocks than SMs.

Tolerance: bf16 outputs within 1e-2 relative L2 of the fp32 reference."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import oracle_sampled, rel_l2

pytestmark = pytest.mark.gpu


def _rand(rng, shape):
    return oracle.round_bf16(rng.uniform(-1, 1, shape).astype(np.float32))


def _check_against_oracle(h, p, a, b, solver, kernel_prefix, variant_has=None):
    got = h.conv_run(p, solver, a, b)
    kern = h.last_kernel()
    assert kern.startswith(kernel_prefix), kern
    if variant_has:
        assert variant_has in h.last_variant(), h.last_variant()
    g, want = oracle_sampled(p, a, b, got)
    err = rel_l2(g, want)
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
    # oracle: f64 direct formula + bias + ReLU on sampled coordinates
    p = problem(n=n, c=c, h=hw, w=hw, k=k)
    rng = np.random.default_rng(7)
    idx = np.stack([rng.integers(0, m, 4096) for m in out.shape], 1)
    from conftest import nchw_to_dev
    acc = oracle.sample_forward(p, nchw_to_dev(x), nchw_to_dev(w), idx, bf16=False)
    want = np.maximum(acc + bias[idx[:, 1]], 0)
    assert rel_l2(out[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]], want) <= 1e-2


def test_pair_gemm_backward_data(lib):
    rng = np.random.default_rng(72)
    p = problem(n=8, c=256, h=56, w=56, k=512, direction=abi.BACKWARD_DATA, etype=abi.BF16)
    sa, sb, _ = operand_shapes(lib, p)
    h = lib.handle()
    _check_against_oracle(h, p, _rand(rng, sa), _rand(rng, sb), "Im2colGemm", "igemm_tc_dgrad")
    print(h.last_variant())


def test_pair_rectangle_stride2_forward(lib):
    rng = np.random.default_rng(73)
    p = problem(n=128, c=256, h=28, w=28, k=256, y=3, x=3, pad=1, stride=2, etype=abi.BF16)
    sa, sb, _ = operand_shapes(lib, p)
    h = lib.handle()
    _check_against_oracle(h, p, _rand(rng, sa), _rand(rng, sb), "ImplicitGemm", "igemm_tc_fwd")
    print(h.last_variant())


@pytest.mark.parametrize("shape", [dict(c=256, k=256, h=14), dict(c=512, k=512, h=7)])
def test_pair_rectangle_backward_data(lib, shape):
    """CTA-pair rectangle dgrad (3x3 stride 1, the conv4_xb / conv5_xb shape)
    at a batch where the grid engages pairs (>= 74 pair tiles)."""
    rng = np.random.default_rng(75)
    p = problem(n=256, y=3, x=3, pad=1, w=shape["h"], direction=abi.BACKWARD_DATA, etype=abi.BF16,
                **shape)
    sa, sb, _ = operand_shapes(lib, p)
    h = lib.handle()
    _check_against_oracle(h, p, _rand(rng, sa), _rand(rng, sb), "Im2colGemm", "igemm_tc_dgrad")
    print(h.last_variant())


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
