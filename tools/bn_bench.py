"""Batch-norm (training) device throughput at ResNet-50 N=256 shapes (BASELINE
cfg4): every distinct BN input shape [256, K, P, P] (bf16, NHWC), timed with
CUDA events on the launching stream, L2 flushed by READING a 512 MB buffer before each
timed call, median of 10. Reports achieved HBM GB/s from algorithmic bytes:
  forward  train: 3 |x| (statistics read, normalise read, y write)
  backward      : 5 |x| (x, dy read for the sums; x, dy read and dx write;
                  no ReLU, i.e. the reference's batchnorm_backward)
and the same for the conv-epilogue variants' finishing passes (bn_finalize_apply:
2 |x|, bn_bwd_finalize_apply: 3 |x| + the ReLU-mask input). Output: one JSON per
line + a summary line (weighted by the 53 layers)."""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import library  # noqa: E402
from paper_1910_00078_b200.resnet50 import resnet50_layers  # noqa: E402

N = int(os.environ.get("BN_N", "256"))
lib = library()
stream = torch.cuda.current_stream()
h = C.c_void_p()
lib.check(lib.lib.primkit_handle_create_with_stream(C.c_void_p(stream.cuda_stream), 0, C.byref(h)))
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0


def timed(fn, reps=int(os.environ.get("BN_REPS", "10"))):
    fn()
    ts = []
    for _ in range(reps):
        flush.max()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
shapes = {}
for L in resnet50_layers():
    shapes[(L.k, L.out_h)] = shapes.get((L.k, L.out_h), 0) + 1
rows = []
tot = {"fwd": [0.0, 0.0], "bwd": [0.0, 0.0]}
for (k, p), count in sorted(shapes.items()):
    x = (torch.rand((N, p, p, k), device="cuda") * 2 - 1).to(torch.bfloat16)
    y, dy, dx = torch.empty_like(x), (torch.rand_like(x, dtype=torch.float32) * 2 - 1).to(torch.bfloat16), \
        torch.empty_like(x)
    g = torch.rand(k, device="cuda") + 0.5
    b = torch.rand(k, device="cuda") - 0.5
    rm, rv = torch.zeros(k, device="cuda"), torch.ones(k, device="cuda")
    sm, si = torch.empty(k, device="cuda"), torch.empty(k, device="cuda")
    dg, db = torch.empty(k, device="cuda"), torch.empty(k, device="cuda")
    dims = (C.c_int64 * 4)(N, k, p, p)
    xb = x.numel() * 2

    def fwd():
        lib.check(lib.lib.primkit_batchnorm_forward_train_device(h, dims, abi.BF16, P(x), P(g), P(b), P(rm), P(rv),
                                                                 C.c_float(1e-5), C.c_float(0.1), P(y), P(sm),
                                                                 P(si), 1))

    def bwd():
        lib.check(lib.lib.primkit_batchnorm_backward_device(h, dims, abi.BF16, P(x), P(y), P(dy), P(g), P(b),
                                                            P(sm), P(si), P(dx), P(dg), P(db), 0))
    fwd()
    tf, tb = timed(fwd), timed(bwd)
    r = {"k": k, "p": p, "layers": count, "mb": xb / 1e6, "fwd_ms": tf, "fwd_gbs": 3 * xb / tf / 1e6,
         "bwd_ms": tb, "bwd_gbs": 5 * xb / tb / 1e6}
    r["fwd_frac"], r["bwd_frac"] = r["fwd_gbs"] / peak, r["bwd_gbs"] / peak
    rows.append(r)
    print(json.dumps(r), flush=True)
    tot["fwd"][0] += count * tf
    tot["fwd"][1] += count * 3 * xb
    tot["bwd"][0] += count * tb
    tot["bwd"][1] += count * 5 * xb
    del x, y, dy, dx
summary = {"summary": True, "n": N, "peak_gbs": peak,
           "fwd_ms_53": tot["fwd"][0], "fwd_gbs": tot["fwd"][1] / tot["fwd"][0] / 1e6,
           "bwd_ms_53": tot["bwd"][0], "bwd_gbs": tot["bwd"][1] / tot["bwd"][0] / 1e6}
summary["fwd_frac"], summary["bwd_frac"] = summary["fwd_gbs"] / peak, summary["bwd_gbs"] / peak
print(json.dumps(summary), flush=True)
