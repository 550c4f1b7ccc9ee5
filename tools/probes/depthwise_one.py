"""One depthwise problem (forward, bwd-data, bwd-weights; bf16), for ncu."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1910_00078_b200 import abi, primkit  # noqa: E402

lib = primkit.library()
h = lib.handle()
rng = np.random.default_rng(0)
for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
    p = primkit.problem(n=32, c=96, h=112, w=112, k=96, y=3, x=3, pad=1, groups=96, etype=abi.BF16,
                        direction=d)
    sa, sb, _ = primkit.operand_shapes(lib, p)
    a = rng.uniform(-1, 1, sa).astype(np.float32)
    b = rng.uniform(-1, 1, sb).astype(np.float32)
    h.conv_run(p, "Direct", a, b)
    print(d, h.last_kernel(), h.last_device_ms())
