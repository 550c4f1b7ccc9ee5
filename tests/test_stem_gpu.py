"""Fused narrow-channel (stem) tcgen05 kernels against the oracle: ResNet
conv1 (3 -> 64, 7x7 stride 2 pad 3), VGG conv1_1 (3 -> 64, 3x3 pad 1) and
ragged / dilated / 128-channel variants, forward (ImplicitGemm), backward data
and backward weights (Im2colGemm), plus the fused epilogue through a fusion
plan.
bf16 tolerance 1e-2 relative L2 against the fp32 oracle (north_star)."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu

STEMS = [
    dict(n=2, c=3, h=64, w=64, k=64, y=7, x=7, pad=3, stride=2),     # ResNet conv1 (reduced)
    dict(n=1, c=3, h=224, w=224, k=64, y=7, x=7, pad=3, stride=2),   # ResNet conv1 full size
    dict(n=2, c=3, h=40, w=40, k=64, y=3, x=3, pad=1),               # VGG conv1_1
    dict(n=3, c=3, h=37, w=45, k=64, y=7, x=7, pad=3, stride=2),     # ragged tiles
    dict(n=2, c=1, h=19, w=23, k=128, y=5, x=5, pad=2, stride=1),    # 1 channel, 128 out
    dict(n=2, c=4, h=21, w=21, k=64, y=3, x=3, pad=2, dilation=2),   # dilated
    dict(n=1, c=2, h=30, w=30, k=64, y=5, x=3, pad_h=0, pad_w=1, stride=2),
]


def _inputs(lib, p, rng):
    sa, sb, _ = operand_shapes(lib, p)
    a = oracle.round_bf16(rng.uniform(-1, 1, sa).astype(np.float32))
    b = oracle.round_bf16(rng.uniform(-1, 1, sb).astype(np.float32))
    return a, b


@pytest.mark.parametrize("si", range(len(STEMS)))
@pytest.mark.parametrize("direction", [abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS])
def test_stem_fused(lib, si, direction):
    if direction == abi.FORWARD and STEMS[si].get("dilation", 1) > 1:
        pytest.skip("ImplicitGemm is forward, dilation 1 only (solver.cpp:167-171)")
    rng = np.random.default_rng(300 + si)
    p = problem(**STEMS[si], direction=direction, etype=abi.BF16)
    h = lib.handle()
    a, b = _inputs(lib, p, rng)
    solver = "ImplicitGemm" if direction == abi.FORWARD else "Im2colGemm"
    got = h.conv_run(p, solver, a, b)
    if direction == abi.BACKWARD_DATA and (STEMS[si]["k"] != 64 or STEMS[si].get("dilation", 1) > 1):
        pytest.skip("fused stem dgrad: 64 dY channels, dilation 1")
    assert h.last_kernel().startswith("stem_fused"), h.last_kernel()
    want = {abi.FORWARD: oracle.conv_forward, abi.BACKWARD_DATA: oracle.conv_backward_data,
            abi.BACKWARD_WEIGHTS: oracle.conv_backward_weights}[direction](p, a, b)
    err = rel_l2(got, want)
    assert err <= 1e-2, err
    assert np.array_equal(oracle.round_bf16(got), got)


def test_stem_fused_deterministic(lib):
    rng = np.random.default_rng(7)
    p = problem(**STEMS[0], direction=abi.BACKWARD_WEIGHTS, etype=abi.BF16)
    h = lib.handle()
    a, b = _inputs(lib, p, rng)
    first = h.conv_run(p, "Im2colGemm", a, b)
    for _ in range(3):
        assert np.array_equal(h.conv_run(p, "Im2colGemm", a, b), first)


def test_stem_fused_epilogue(lib):
    """conv + bias + BN(inference) + ReLU on a 3-channel bf16 input: one
    fused stem kernel with the folded per-channel affine epilogue."""
    rng = np.random.default_rng(11)
    n, c, hw, k = 2, 3, 33, 64
    plan = lib.fusion_plan((n, c, hw, hw), abi.BF16)
    lib.check(plan.add_conv((k, c, 3, 3), pad=1))
    lib.check(plan.add_bias(k))
    lib.check(plan.add_batchnorm(abi.BN_SPATIAL))
    lib.check(plan.add_activation(abi.RELU))
    h = lib.handle()
    lib.check(plan.compile(h))
    w = oracle.round_bf16(rng.uniform(-1, 1, (k, c, 3, 3)).astype(np.float32))
    bias = rng.uniform(-1, 1, k).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, k).astype(np.float32)
    beta = rng.uniform(-1, 1, k).astype(np.float32)
    mean = rng.uniform(-1, 1, k).astype(np.float32)
    var = (1 + np.abs(rng.uniform(-1, 1, k))).astype(np.float32)
    plan.set_args(filter=w, bias=bias, gamma=gamma, beta=beta, mean=mean, var=var, eps=1e-5)
    x = oracle.round_bf16(rng.uniform(-1, 1, (n, c, hw, hw)).astype(np.float32))
    got = plan.execute(h, x)
    p = problem(n=n, c=c, h=hw, w=hw, k=k, y=3, x=3, pad=1)
    y = oracle.conv_forward(p, x, w) + bias[None, :, None, None]
    y = (y - mean[None, :, None, None]) / np.sqrt(var[None, :, None, None] + 1e-5) * \
        gamma[None, :, None, None] + beta[None, :, None, None]
    want = np.maximum(y, 0)
    assert rel_l2(got, want) <= 1e-2
