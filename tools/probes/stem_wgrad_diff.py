"""Compare the ResNet conv1 backward-weights kernels (PK_STEM_WG=1 vs 2) per tap:
run with PK_STEM_WG unset (row strips) and =1 in two processes, diff the dumps."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import library, problem  # noqa: E402

n = int(os.environ.get("N", "2"))
lib = library()
h = C.c_void_p()
lib.check(lib.lib.primkit_handle_create_with_stream(C.c_void_p(torch.cuda.current_stream().cuda_stream), 0,
                                                    C.byref(h)))
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.zeros(n, 224, 224, 8, device="cuda", dtype=torch.bfloat16)
x[..., :3] = (torch.rand(n, 224, 224, 3, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
dy = ((torch.rand(n, 112, 112, 64, device="cuda", generator=g) * 2 - 1)).to(torch.bfloat16)
dw = torch.zeros(64, 7, 7, 8, device="cuda", dtype=torch.bfloat16)
p = problem(n=n, c=3, h=224, w=224, k=64, y=7, x=7, pad=3, stride=2, direction=abi.BACKWARD_WEIGHTS,
            etype=abi.BF16)
ws_b = C.c_uint64()
lib.check(lib.lib.primkit_conv_device_workspace(h, C.byref(p), b"Im2colGemm", C.byref(ws_b)))
ws = torch.empty(max(ws_b.value, 256), dtype=torch.uint8, device="cuda")
lib.check(lib.lib.primkit_conv_run_device(h, C.byref(p), b"Im2colGemm", C.c_void_p(dy.data_ptr()),
                                          C.c_void_p(x.data_ptr()), C.c_void_p(dw.data_ptr()),
                                          C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel())))
torch.cuda.synchronize()
# exact reference in fp32 on the GPU (unfold)
xf = x[..., :3].permute(0, 3, 1, 2).float()
dyf = dy.permute(0, 3, 1, 2).float()
ref = torch.nn.grad.conv2d_weight(xf, (64, 3, 7, 7), dyf, stride=2, padding=3)  # [64][3][7][7]
got = dw[..., :3].permute(0, 3, 1, 2).float()
err = (got - ref).abs()
print("rel-L2", float((got - ref).norm() / ref.norm()))
per_r = [(r, float((got[:, :, r] - ref[:, :, r]).norm() / ref[:, :, r].norm())) for r in range(7)]
per_s = [(s, float((got[:, :, :, s] - ref[:, :, :, s]).norm() / ref[:, :, :, s].norm())) for s in range(7)]
per_c = [(c, float((got[:, c] - ref[:, c]).norm() / ref[:, c].norm())) for c in range(3)]
per_kh = [(k0, float((got[k0:k0 + 32] - ref[k0:k0 + 32]).norm() / ref[k0:k0 + 32].norm())) for k0 in (0, 32)]
print("per r", per_r)
print("per s", per_s)
print("per c", per_c)
print("per k half", per_kh)
print("ratio got/ref (r=3,s=3) first k:", (got[:4, 0, 3, 3] / ref[:4, 0, 3, 3]).tolist())
