"""Small invocations of the 64-channel halo kernel (256-position tiles) for
compute-sanitizer: ResNet conv2_x 3x3 geometry at N=2, forward and backward data,
each checked against the oracle."""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import library, problem  # noqa: E402

lib = library()
h = lib.handle()
rng = np.random.default_rng(0)


def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b))


p = problem(n=2, c=64, h=56, w=56, k=64, y=3, x=3, pad=1, etype=abi.BF16)
x = oracle.round_bf16(rng.uniform(-1, 1, (2, 64, 56, 56)).astype(np.float32))
w = oracle.round_bf16(rng.uniform(-1, 1, (64, 64, 3, 3)).astype(np.float32))
y = h.conv_run(p, "ImplicitGemm", x, w)
print("halo fwd", h.last_variant(), rel(y, oracle.conv_forward(p, x, w)))
pd = problem(n=2, c=64, h=56, w=56, k=64, y=3, x=3, pad=1, direction=abi.BACKWARD_DATA, etype=abi.BF16)
dy = oracle.round_bf16(rng.uniform(-1, 1, (2, 64, 56, 56)).astype(np.float32))
dx = h.conv_run(pd, "Im2colGemm", dy, w)
print("halo dgrad", h.last_variant(), rel(dx, oracle.conv_backward_data(pd, dy, w)))
