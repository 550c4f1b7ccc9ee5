"""Time every applicable solver on depthwise / grouped problems (device ms of
the conv itself, `primkit_handle_last_device_ms`), beside the HBM bound of
x + w + y bytes. Run on a GPU box: python tools/probes/depthwise_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1910_00078_b200 import abi, primkit  # noqa: E402

lib = primkit.library()
h = lib.handle()
rng = np.random.default_rng(0)
cases = [dict(n=32, c=96, h=112, w=112, k=96, y=3, x=3, pad=1, groups=96),
         dict(n=64, c=256, h=28, w=28, k=256, y=3, x=3, pad=1, groups=256),
         dict(n=64, c=256, h=28, w=28, k=256, y=3, x=3, pad=1, groups=32)]
for cs in cases:
    for et, esz in ((abi.BF16, 2), (abi.F32, 4)):
        for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
            p = primkit.problem(**cs, etype=et, direction=d)
            sa, sb, so = primkit.operand_shapes(lib, p)
            a = rng.uniform(-1, 1, sa).astype(np.float32)
            b = rng.uniform(-1, 1, sb).astype(np.float32)
            byts = (np.prod(sa) + np.prod(sb) + np.prod(so)) * esz
            for s in h.solver_names():
                if not h.is_applicable(s, p):
                    continue
                ms = []
                for _ in range(3):
                    h.conv_run(p, s, a, b)
                    ms.append(h.last_device_ms())
                print(f"{cs['groups']:4d} {cs['c']}x{cs['h']} {'bf16' if et == abi.BF16 else 'f32 '} "
                      f"dir={d} {s:14s} {min(ms):8.3f} ms  hbm {byts / 6.55e9:6.3f} ms  "
                      f"{h.last_kernel()}", flush=True)
