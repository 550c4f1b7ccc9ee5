"""Where the host-buffer (primkit_conv_run) step time goes: wall time per
direction vs its PCIe byte bound (H2D and D2H at the measured link rates)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import library, operand_shapes, problem  # noqa: E402
from paper_1910_00078_b200.resnet50 import resnet50_layers  # noqa: E402

lib = library()
h = C.c_void_p()
lib.check(lib.lib.primkit_handle_create(C.byref(h)))
n = 256
calls = {0: [], 1: [], 2: []}
max_el = 0
for L in resnet50_layers():
    for d, s in ((abi.FORWARD, "ImplicitGemm"), (abi.BACKWARD_DATA, "Im2colGemm"),
                 (abi.BACKWARD_WEIGHTS, "Im2colGemm")):
        p = problem(n=n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad, stride=L.stride,
                    direction=d, etype=abi.BF16)
        sa, sb, so = operand_shapes(lib, p)
        na, nb, no = (int(np.prod(v)) for v in (sa, sb, so))
        max_el = max(max_el, na, nb, no)
        calls[d].append((L.name, p, s.encode(), na, nb, no))
bufs = [torch.empty(max_el, dtype=torch.float32).pin_memory() for _ in range(3)]
for b in bufs:
    b.uniform_(-1, 1)
ptrs = [C.cast(C.c_void_p(b.data_ptr()), C.POINTER(C.c_float)) for b in bufs]
ws = C.c_size_t(1 << 34)
for d in (0, 1, 2):
    for (_, p, s, na, nb, no) in calls[d]:
        lib.check(lib.lib.primkit_conv_run(h, C.byref(p), s, ptrs[0], ptrs[1], ptrs[2], ws))
H2D, D2H = 55.6e9, 57.2e9
tot = 0.0
for d in (0, 1, 2):
    rows = []
    t_all = 0.0
    for (name, p, s, na, nb, no) in calls[d]:
        t0 = time.perf_counter()
        lib.check(lib.lib.primkit_conv_run(h, C.byref(p), s, ptrs[0], ptrs[1], ptrs[2], ws))
        t = time.perf_counter() - t0
        t_all += t
        bound = max(4 * (na + nb) / H2D, 4 * no / D2H)
        rows.append((t, bound, name))
    tot += t_all
    b_all = sum(r[1] for r in rows)
    print(f"dir {d}: wall {t_all * 1e3:.1f} ms, per-call byte bound {b_all * 1e3:.1f} ms "
          f"({b_all / t_all:.2f})")
    for t, b, name in sorted(rows, key=lambda r: -(r[0] - r[1]))[:5]:
        print(f"   {name:>10} {t * 1e3:7.2f} ms bound {b * 1e3:6.2f}")
print(f"step {tot * 1e3:.1f} ms")
