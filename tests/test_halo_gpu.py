"""Halo-reuse tcgen05 path (conv_halo.cu) for stride-1 spatial filters:
forward (ImplicitGemm) and backward data (Im2colGemm) against the oracle on
shapes that exercise ragged grid rows, padding 0/1/2, 5x5 taps, two input
chunks and a 256-wide output tile (bf16 tolerance 1e-2 relative L2)."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu

HALO = [
    dict(n=2, c=64, h=56, w=56, k=64, y=3, x=3, pad=1),     # ResNet conv2_x 3x3
    dict(n=2, c=64, h=30, w=33, k=128, y=3, x=3, pad=1),    # ragged rows, N=128
    dict(n=1, c=128, h=28, w=28, k=256, y=3, x=3, pad=1),   # 2 chunks, N=256
    dict(n=1, c=64, h=48, w=48, k=64, y=5, x=5, pad=2),     # 5x5
    dict(n=2, c=64, h=40, w=40, k=64, y=3, x=3, pad=0),     # no padding
    dict(n=1, c=64, h=44, w=44, k=192, y=3, x=3, pad=1),    # N not a power of two
]


@pytest.mark.parametrize("si", range(len(HALO)))
@pytest.mark.parametrize("direction", [abi.FORWARD, abi.BACKWARD_DATA])
def test_halo_conv(lib, si, direction):
    rng = np.random.default_rng(900 + si)
    p = problem(**HALO[si], direction=direction, etype=abi.BF16)
    sa, sb, _ = operand_shapes(lib, p)
    a = oracle.round_bf16(rng.uniform(-1, 1, sa).astype(np.float32))
    b = oracle.round_bf16(rng.uniform(-1, 1, sb).astype(np.float32))
    h = lib.handle()
    solver = "ImplicitGemm" if direction == abi.FORWARD else "Im2colGemm"
    got = h.conv_run(p, solver, a, b)
    want = (oracle.conv_forward(p, a, b) if direction == abi.FORWARD
            else oracle.conv_backward_data(p, a, b))
    assert rel_l2(got, want) <= 1e-2
    assert np.array_equal(oracle.round_bf16(got), got)
