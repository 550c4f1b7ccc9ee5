"""Fused vs unfused conv+bias+ReLU (cfg2 shape) through the device fusion API;
target of the ncu launch-list capture in profiles/."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import library  # noqa: E402

lib = library()
h = C.c_void_p()
lib.check(lib.lib.primkit_handle_create_with_stream(
    C.c_void_p(torch.cuda.current_stream().cuda_stream), 0, C.byref(h)))


class H:
    ptr = h


n, c, k, hw, f, pad = 64, 64, 256, 56, 1, 0
if len(sys.argv) > 1 and sys.argv[1] == "3x3":
    k, f, pad = 64, 3, 1
plan = lib.fusion_plan((n, c, hw, hw), abi.BF16)
lib.check(plan.add_conv((k, c, f, f), pad=pad))
lib.check(plan.add_bias(k))
if f == 3:
    lib.check(plan.add_batchnorm(abi.BN_SPATIAL))
lib.check(plan.add_activation(abi.RELU))
lib.check(plan.compile(H()))
rng = np.random.default_rng(0)
plan.set_args(filter=rng.uniform(-1, 1, (k, c, f, f)).astype(np.float32),
              bias=rng.uniform(-1, 1, k).astype(np.float32), gamma=np.ones(k, np.float32),
              beta=np.zeros(k, np.float32), mean=np.zeros(k, np.float32), var=np.ones(k, np.float32))
x = (torch.rand((n, hw, hw, c), device="cuda") * 2 - 1).to(torch.bfloat16)
y = torch.empty((n, hw, hw, k), device="cuda", dtype=torch.bfloat16)
for unf in (0, 1, 0, 1):
    lib.check(lib.lib.primkit_fusion_execute_device(h, plan.ptr, C.c_void_p(x.data_ptr()),
                                                    C.c_void_p(y.data_ptr()), unf))
torch.cuda.synchronize()
print("done")
