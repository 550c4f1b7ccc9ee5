"""One eager ResNet-50 conv step (53 layers x fwd/bwdData/bwdWeights, bf16,
N=256) after one warm-up step; target of the ncu launch-list capture."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1910_00078_b200.primkit import library  # noqa: E402
from paper_1910_00078_b200.resnet50 import resnet50_layers  # noqa: E402

lib = library()
h = C.c_void_p()
lib.check(lib.lib.primkit_handle_create_with_stream(
    C.c_void_p(torch.cuda.current_stream().cuda_stream), 0, C.byref(h)))


class H:
    ptr = h


net = bench.Net(torch, lib, H(), resnet50_layers(), int(os.environ.get("PK_BATCH", "256")),
                torch.device("cuda", 0))
bench.step(lib, H(), net)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
bench.step(lib, H(), net)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("step done")
