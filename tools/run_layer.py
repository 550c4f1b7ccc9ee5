"""Run one ResNet-50 layer (fwd/bwd_data/bwd_weights) through the device API a
few times; used as the target of ncu captures (profiles/)."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import library, problem  # noqa: E402
from paper_1910_00078_b200.resnet50 import resnet50_layers  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layer", default="conv4_2b")
ap.add_argument("--dir", type=int, default=0)
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--time", action="store_true", help="print the mean CUDA-event time per call")
a = ap.parse_args()
L = {l.name: l for l in resnet50_layers()}[a.layer]
lib = library()
h = C.c_void_p()
lib.check(lib.lib.primkit_handle_create_with_stream(
    C.c_void_p(torch.cuda.current_stream().cuda_stream), 0, C.byref(h)))
cp, kp = lib.channel_pitch(L.c), lib.channel_pitch(L.k)
ho = L.out_h
x = torch.randn(a.n, L.h, L.h, cp, device="cuda").to(torch.bfloat16)
w = torch.randn(L.k, L.r, L.r, cp, device="cuda").to(torch.bfloat16)
y = torch.randn(a.n, ho, ho, kp, device="cuda").to(torch.bfloat16)
solver = b"ImplicitGemm" if a.dir == 0 else b"Im2colGemm"
p = problem(n=a.n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad, stride=L.stride,
            direction=a.dir, etype=abi.BF16)
ws_b = C.c_uint64()
lib.check(lib.lib.primkit_conv_device_workspace(h, C.byref(p), solver, C.byref(ws_b)))
ws = torch.empty(max(ws_b.value, 256), dtype=torch.uint8, device="cuda")
ops = {0: (x, w, y), 1: (y, w, x), 2: (y, x, w)}[a.dir]
def call():
    lib.check(lib.lib.primkit_conv_run_device(h, C.byref(p), solver, C.c_void_p(ops[0].data_ptr()),
                                              C.c_void_p(ops[1].data_ptr()),
                                              C.c_void_p(ops[2].data_ptr()),
                                              C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel())))


for _ in range(a.iters):
    call()
torch.cuda.synchronize()
if a.time:
    # device time without host launch overhead (as bench.py's layer report): 10 calls in a graph
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        lib.check(lib.lib.primkit_handle_set_stream(h, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        for _ in range(10):
            call()
    lib.check(lib.lib.primkit_handle_set_stream(h, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{a.layer} dir {a.dir} N={a.n} env={os.environ.get('PK_STEM_DEBUG', '')}/{os.environ.get('PK_STEM_DG', '')}: "
          f"{e0.elapsed_time(e1) / 30 * 1e3:.1f} us")
print("done", a.layer, a.dir)
