"""Time every applicable solver on transpose-mode, dilated and FFT-sized problems
(device ms of the conv itself). Run on a GPU box: python tools/probes/modes_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1910_00078_b200 import abi, primkit  # noqa: E402

lib = primkit.library()
h = lib.handle()
rng = np.random.default_rng(0)
cases = [("transpose 3x3 s2", dict(n=32, c=256, h=28, w=28, k=128, y=3, x=3, pad=1, stride=2,
                                   mode=abi.TRANSPOSE)),
         ("dilated 3x3 d2", dict(n=32, c=256, h=28, w=28, k=256, y=3, x=3, pad=2, dilation=2)),
         ("plain 5x5", dict(n=32, c=64, h=56, w=56, k=64, y=5, x=5, pad=2))]
for name, cs in cases:
    for et in (abi.BF16, abi.F32):
        for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
            p = primkit.problem(**cs, etype=et, direction=d)
            sa, sb, so = primkit.operand_shapes(lib, p)
            a = rng.uniform(-1, 1, sa).astype(np.float32)
            b = rng.uniform(-1, 1, sb).astype(np.float32)
            for s in h.solver_names():
                if not h.is_applicable(s, p):
                    continue
                ms = []
                for _ in range(2):
                    h.conv_run(p, s, a, b)
                    ms.append(h.last_device_ms())
                print(f"{name:18s} {'bf16' if et == abi.BF16 else 'f32 '} dir={d} {s:13s} {min(ms):9.3f} ms "
                      f"{h.last_kernel()}", flush=True)
