"""Device time of the FFT solver (and Direct for comparison) on a 5x5 64ch 56x56
N=32 fp32 forward, the shape of profiles/r01_simt_paths.txt."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1910_00078_b200.primkit import library, problem  # noqa: E402

lib = library()
h = C.c_void_p()
lib.check(lib.lib.primkit_handle_create_with_stream(C.c_void_p(torch.cuda.current_stream().cuda_stream), 0,
                                                    C.byref(h)))
n, c, hw, k, r = 32, 64, 56, 64, 5
p = problem(n=n, c=c, h=hw, w=hw, k=k, y=r, x=r, pad=2)
x = torch.rand(n, hw, hw, c, device="cuda") * 2 - 1
w = torch.rand(k, r, r, c, device="cuda") * 2 - 1
for solver in (b"FFT", b"Direct", b"ImplicitGemm"):
    y = torch.empty(n, hw, hw, k, device="cuda")
    ws_b = C.c_uint64()
    lib.check(lib.lib.primkit_conv_device_workspace(h, C.byref(p), solver, C.byref(ws_b)))
    ws = torch.empty(max(ws_b.value, 256), dtype=torch.uint8, device="cuda")

    def call():
        lib.check(lib.lib.primkit_conv_run_device(h, C.byref(p), solver, C.c_void_p(x.data_ptr()),
                                                  C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr()),
                                                  C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel())))
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        call()
    e1.record()
    torch.cuda.synchronize()
    kn = C.create_string_buffer(64)
    lib.lib.primkit_handle_last_kernel(h, kn, 64)
    print(solver.decode(), kn.value.decode(), f"{e0.elapsed_time(e1) / 5:.3f} ms", f"ws {ws_b.value / 1e6:.0f} MB")
