"""Small invocations of the round-2 kernels for compute-sanitizer: the stem row-strip
forward / backward-data kernels (ResNet conv1 geometry at 64x64) and the 3xTF32 fp32
forward, each checked against the oracle."""
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


p = problem(n=2, c=3, h=64, w=64, k=64, y=7, x=7, pad=3, stride=2, etype=abi.BF16)
x = oracle.round_bf16(rng.uniform(-1, 1, (2, 3, 64, 64)).astype(np.float32))
w = oracle.round_bf16(rng.uniform(-1, 1, (64, 3, 7, 7)).astype(np.float32))
y = h.conv_run(p, "ImplicitGemm", x, w)
print("stem fwd", h.last_variant(), rel(y, oracle.conv_forward(p, x, w)))
pd = problem(n=2, c=3, h=64, w=64, k=64, y=7, x=7, pad=3, stride=2, direction=abi.BACKWARD_DATA,
             etype=abi.BF16)
dy = oracle.round_bf16(rng.uniform(-1, 1, (2, 64, 32, 32)).astype(np.float32))
dx = h.conv_run(pd, "Im2colGemm", dy, w)
print("stem dgrad", h.last_variant(), rel(dx, oracle.conv_backward_data(pd, dy, w)))
pf = problem(n=2, c=64, h=8, w=8, k=64, y=3, x=3, pad=1)
xf = rng.uniform(-1, 1, (2, 64, 8, 8)).astype(np.float32)
wf = rng.uniform(-1, 1, (64, 64, 3, 3)).astype(np.float32)
yf = h.conv_run(pf, "ImplicitGemm", xf, wf)
print("tf32x3", h.last_kernel(), rel(yf, oracle.conv_forward(pf, xf, wf)))
