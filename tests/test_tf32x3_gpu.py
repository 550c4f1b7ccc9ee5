"""fp32 forward convolutions on the tensor cores at fp32 accuracy (3xTF32).

Direct / ImplicitGemm / Im2colGemm fp32 forward problems with groups 1 and a channel pitch
that is a multiple of 32 run `tf32x3_tc_fwd`: the operands are split into a
tf32 "hi" part and an fp32 remainder "lo" (conv_tma.cu tf32x3_split_kernel) and
one tcgen05 kind::tf32 GEMM over the concatenation sums hi.hi + hi.lo + lo.hi.
The north_star tolerance for fp32 is 1e-4 relative L2 against the CPU oracle
(proj/src/core/conv.cpp direct_forward); the reference's own max-rel metric is
checked too. Fused conv+bias+ReLU on the Direct row goes the same way
(fusion.cpp), with the reference epilogue formula before the fp32 store."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import problem

from conftest import max_rel, rel_l2

pytestmark = pytest.mark.gpu

SHAPES = [
    dict(n=2, c=64, h=8, w=8, k=64, y=3, x=3, pad=1),                  # ResNet conv2_x 3x3
    dict(n=1, c=32, h=9, w=9, k=48, y=1, x=1, stride=2),               # strided 1x1, ragged K
    dict(n=2, c=32, h=13, w=11, k=96, y=5, x=5, pad=2),                # 5x5, ragged tiles
    dict(n=1, c=32, h=12, w=12, k=32, y=3, x=3, pad=0, dilation=2),    # dilated
    dict(n=3, c=128, h=7, w=7, k=256, y=1, x=1),                       # wide 1x1
    dict(n=1, c=64, h=15, w=15, k=64, y=3, x=3, pad=1, stride=2),      # strided 3x3
]


@pytest.mark.parametrize("si", range(len(SHAPES)))
@pytest.mark.parametrize("solver", ["ImplicitGemm", "Direct", "Im2colGemm"])
def test_tf32x3_forward_matches_fp32_oracle(lib, si, solver):
    rng = np.random.default_rng(500 + si)
    sh = SHAPES[si]
    if solver == "ImplicitGemm" and sh.get("dilation", 1) > 1:
        pytest.skip("ImplicitGemm rejects dilation (proj/src/core/solver.cpp:167-171)")
    p = problem(**sh)
    x = rng.uniform(-1, 1, (sh["n"], sh["c"], sh["h"], sh["w"])).astype(np.float32)
    w = rng.uniform(-1, 1, (sh["k"], sh["c"], sh["y"], sh["x"])).astype(np.float32)
    h = lib.handle()
    got = h.conv_run(p, solver, x, w)
    assert h.last_kernel() == "tf32x3_tc_fwd", h.last_kernel()
    want = oracle.conv_forward(p, x, w)
    assert rel_l2(got, want) <= 1e-4, rel_l2(got, want)
    assert max_rel(got, want) <= 1e-4


def test_tf32x3_beats_single_tf32_rounding(lib):
    # one tf32 pass would leave ~1e-3 relative errors on large-magnitude sums; the
    # split keeps the error at fp32 level
    rng = np.random.default_rng(7)
    p = problem(n=2, c=128, h=6, w=6, k=64, y=3, x=3, pad=1)
    x = (rng.uniform(-1, 1, (2, 128, 6, 6)) * 1000).astype(np.float32)
    w = rng.uniform(-1, 1, (64, 128, 3, 3)).astype(np.float32)
    h = lib.handle()
    got = h.conv_run(p, "ImplicitGemm", x, w)
    want = oracle.conv_forward(p, x, w)
    assert rel_l2(got, want) <= 1e-5


def test_tf32x3_deep_reductions_stay_on_fma(lib):
    # R*S*C above 1152: the tensor core's accumulation error would exceed the
    # reference's max-rel 1e-4, so the fp32 FMA kernel runs
    p = problem(n=1, c=64, h=9, w=9, k=32, y=5, x=5, pad=2)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (1, 64, 9, 9)).astype(np.float32)
    w = rng.uniform(-1, 1, (32, 64, 5, 5)).astype(np.float32)
    h = lib.handle()
    got = h.conv_run(p, "ImplicitGemm", x, w)
    assert h.last_kernel() != "tf32x3_tc_fwd", h.last_kernel()
    assert max_rel(got, oracle.conv_forward(p, x, w)) <= 1e-4


def test_tf32x3_fused_bias_relu(lib):
    rng = np.random.default_rng(11)
    n, c, hw, k = 2, 64, 10, 64
    plan = lib.fusion_plan((n, c, hw, hw), abi.F32)
    lib.check(plan.add_conv((k, c, 1, 1)))
    lib.check(plan.add_bias(k))
    lib.check(plan.add_activation(abi.RELU))
    h = lib.handle()
    lib.check(plan.compile(h))
    wf = rng.uniform(-1, 1, (k, c, 1, 1)).astype(np.float32)
    b = rng.uniform(-1, 1, k).astype(np.float32)
    xf = rng.uniform(-1, 1, (n, c, hw, hw)).astype(np.float32)
    plan.set_args(filter=wf, bias=b)
    out = plan.execute(h, xf)
    assert h.last_kernel() == "tf32x3_tc_fwd+epilogue", h.last_kernel()
    pf = problem(n=n, c=c, h=hw, w=hw, k=k)
    ref = np.maximum(oracle.conv_forward(pf, xf, wf) + b[None, :, None, None], 0)
    assert rel_l2(out, ref) <= 1e-4
