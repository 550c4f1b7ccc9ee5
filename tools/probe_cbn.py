"""Per-layer breakdown of the conv+BN paths (profiling helper)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools.bench_configs import Dev, timed, vp  # noqa: E402
from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import problem  # noqa: E402
from paper_1910_00078_b200.resnet50 import resnet50_layers  # noqa: E402

d = Dev()
lib = d.lib
n = 256
for name in sys.argv[1:] or ["conv2_1c", "conv3_2b", "conv4_2a", "conv1"]:
    L = {l.name: l for l in resnet50_layers()}[name]
    ho = L.out_h
    p = problem(n=n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad, stride=L.stride, etype=abi.BF16)
    x, w = d.act(n, L.h, L.h, L.c, torch.bfloat16), d.act(L.k, L.r, L.r, L.c, torch.bfloat16)
    kp = lib.channel_pitch(L.k)
    conv = torch.empty((n, ho, ho, kp), device="cuda", dtype=torch.bfloat16)
    z = torch.empty_like(conv)
    vec = lambda v: torch.full((L.k,), v, device="cuda")  # noqa: E731
    g, b, rm, rv, sm, si = vec(1.0), vec(0.0), vec(0.0), vec(1.0), vec(0.0), vec(1.0)
    ws = d.ws(p, b"ImplicitGemm", "primkit_conv_bn_workspace")
    dims = (C.c_int64 * 4)(n, L.k, ho, ho)
    t_conv = timed(lambda: d.conv(p, b"ImplicitGemm", x, w, conv, ws), 10)
    t_bn = timed(lambda: lib.check(lib.lib.primkit_batchnorm_forward_train_device(
        d.h, dims, abi.BF16, vp(conv), vp(g), vp(b), vp(rm), vp(rv), C.c_float(1e-5),
        C.c_float(0.1), vp(z), vp(sm), vp(si), 1)), 10)
    t_fused = timed(lambda: lib.check(lib.lib.primkit_conv_bn_forward_train_device(
        d.h, C.byref(p), b"ImplicitGemm", vp(x), vp(w), vp(g), vp(b), vp(rm), vp(rv),
        C.c_float(1e-5), C.c_float(0.1), vp(conv), vp(z), vp(sm), vp(si), 1, vp(ws),
        C.c_size_t(ws.numel()))), 10)
    mb = conv.numel() * 2 / 1e6
    print(f"{name}: conv {t_conv:.3f} ms, standalone BN {t_bn:.3f} ms ({3 * mb / t_bn / 1e3:.0f} GB/s eff), "
          f"fused conv+BN {t_fused:.3f} ms; y {mb:.0f} MB")
