"""Narrow-tile paths of the tcgen05 kernels at sizes where every CTA owns
several tiles, against the oracle (bf16 <= 1e-2 relative L2):

* conv_tc_kernel with BN <= 64 splits its epilogue by TILE over four TMEM
  accumulator buffers (conv_tc.cu kSplit); the strided 1x1 backward-data case
  also has tap-less sub-pixel phases whose zero tiles go to one epilogue half;
* gemm_pair_kernel runs the last partial round of pair tiles as half tiles
  (conv_tc2.cu pair_item) when 2 * (tiles mod pairs) <= pairs.
The full-size ResNet-50 instances of both are in test_step_parity_gpu.py."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu

CASES = [
    # 1x1 stride 2, dx with 32 channels: PHASE_DGRAD, BN = 32, 3 of 4 phases tap-less
    ("dgrad_1x1_s2_c32", dict(n=32, c=32, h=56, w=56, k=64, y=1, x=1, stride=2), abi.BACKWARD_DATA,
     "conv_tc_kernel<32"),
    # 3x3 on 32 channels (pitch not a multiple of 64): gather modes, BN = 64
    ("fwd_3x3_c32_k64", dict(n=16, c=32, h=28, w=28, k=64, y=3, x=3, pad=1), abi.FORWARD,
     "conv_tc_kernel<64"),
    # (its backward data runs the 64-wide TMA rectangle kernel on a transposed filter)
    ("dgrad_3x3_c64_k32", dict(n=16, c=64, h=28, w=28, k=32, y=3, x=3, pad=1), abi.BACKWARD_DATA,
     "conv_tma_fprop_kernel<64"),
    # 1x1 64 -> 64 plain GEMM with the resident filter, BN = 64
    ("fwd_1x1_c64_k64", dict(n=16, c=64, h=28, w=28, k=64, y=1, x=1), abi.FORWARD,
     "conv_tc_kernel<64"),
    # pair GEMM: M = 160*7*7 = 7840 -> 31 M pairs x 4 N tiles = 124 tiles on 74 pairs:
    # 50 left, 100 halves > 74 -> whole tiles only
    ("fwd_1x1_pair_small", dict(n=160, c=512, h=7, w=7, k=1024, y=1, x=1), abi.FORWARD, "gemm_pair"),
    # M = 256*7*7 = 12544 -> 49 M pairs x 2 N tiles = 98 tiles: 24 left -> 48 half tiles
    ("fwd_1x1_pair_tail", dict(n=256, c=512, h=7, w=7, k=512, y=1, x=1), abi.FORWARD, "gemm_pair"),
    ("dgrad_1x1_pair_tail", dict(n=256, c=512, h=7, w=7, k=512, y=1, x=1), abi.BACKWARD_DATA,
     "gemm_pair"),
]


@pytest.mark.parametrize("name,shape,direction,variant", CASES, ids=[c[0] for c in CASES])
def test_narrow_and_tail_tiles(lib, name, shape, direction, variant):
    rng = np.random.default_rng(7)
    p = problem(**shape, direction=direction, etype=abi.BF16)
    sa, sb, _ = operand_shapes(lib, p)
    a = oracle.round_bf16(rng.uniform(-1, 1, sa).astype(np.float32))
    b = oracle.round_bf16(rng.uniform(-1, 1, sb).astype(np.float32))
    want = oracle.conv_forward(p, a, b) if direction == abi.FORWARD else oracle.conv_backward_data(p, a, b)
    h = lib.handle()
    got = h.conv_run(p, "ImplicitGemm" if direction == abi.FORWARD else "Im2colGemm", a, b)
    err = rel_l2(got, want)
    assert err <= 1e-2, f"{name}: {h.last_kernel()} rel-L2 {err:.3e}"
    assert np.array_equal(oracle.round_bf16(got), got)
    assert variant in h.last_variant(), f"{name} ran {h.last_variant()}"
