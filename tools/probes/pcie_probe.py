"""PCIe and host-conversion rates on the GPU box (calibrates the host-ABI
pipeline): pinned H2D, D2H, both directions concurrently, and the host-side
f32 -> bf16 conversion throughput with torch's CPU threads."""
import time

import torch

n = 256 * 1024 * 1024  # 1 GiB of f32
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


gb = n * 4 / 1e9
th2d = t(lambda: d.copy_(h, non_blocking=True))
td2h = t(lambda: h.copy_(d, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


tb = t(both)
print(f"H2D {gb / th2d:.1f} GB/s, D2H {gb / td2h:.1f} GB/s, concurrent {2 * gb / tb:.1f} GB/s total")
x = torch.rand(n)
for th in (1, 4, 8, 16, 32):
    torch.set_num_threads(th)
    tc = t(lambda: x.to(torch.bfloat16), 2)
    print(f"host f32->bf16 with {th} threads: {gb / tc:.1f} GB/s of f32 input")
import os
print("cpus", os.cpu_count())
