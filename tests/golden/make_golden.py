"""Generate tests/golden/*.npz from the UNMODIFIED reference implementation
(oracle/_ref/libprimkit_ref.so, compiled from /root/reference sources by
oracle/Makefile.ref). Run here (where the reference sources exist):

    python tests/golden/make_golden.py

The fixtures pin the oracle restatement and the GPU path on boxes where the
reference cannot be rebuilt. Inputs are seeded U(-1, 1) (bf16 cases rounded
with the reference's own round_bf16)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import operand_shapes, problem  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CONV_CASES = [
    ("fwd_3x3_p1", dict(n=2, c=4, h=8, w=8, k=4, y=3, x=3, pad=1), abi.FORWARD),
    ("fwd_7x7_s2", dict(n=1, c=3, h=13, w=13, k=8, y=7, x=7, pad=3, stride=2), abi.FORWARD),
    ("fwd_dil2_g2", dict(n=2, c=4, h=9, w=9, k=6, y=3, x=3, pad=1, dilation=2, groups=2),
     abi.FORWARD),
    ("bd_3x3_s2", dict(n=2, c=6, h=9, w=9, k=4, y=3, x=3, pad=1, stride=2), abi.BACKWARD_DATA),
    ("bw_3x3_p1", dict(n=2, c=5, h=7, w=7, k=3, y=3, x=3, pad=1), abi.BACKWARD_WEIGHTS),
    ("bw_1x1_s2", dict(n=3, c=8, h=6, w=6, k=4, y=1, x=1, stride=2), abi.BACKWARD_WEIGHTS),
]


def main():
    ref = oracle.reference()
    if ref is None:
        oracle.build()
        ref = oracle.reference()
    h = ref.handle()
    rng = np.random.default_rng(20261017)
    data = {}
    for name, shp, d in CONV_CASES:
        for et in (abi.F32, abi.BF16):
            p = problem(**shp, direction=d, etype=et)
            sa, sb, _ = operand_shapes(ref, p)
            a = rng.uniform(-1, 1, sa).astype(np.float32)
            b = rng.uniform(-1, 1, sb).astype(np.float32)
            if et == abi.BF16:
                a, b = oracle.round_bf16(a), oracle.round_bf16(b)
            tag = f"{name}_{'bf16' if et else 'f32'}"
            data[tag + "_a"] = a
            data[tag + "_b"] = b
            data[tag + "_direct"] = h.conv_run(p, "Direct", a, b)
            if d == abi.FORWARD and shp["y"] == 3 and shp.get("stride", 1) == 1 and \
                    shp.get("dilation", 1) == 1:
                data[tag + "_winograd"] = h.conv_run(p, "Winograd", a, b)
    # batch-norm, spatial and per-activation
    for mode in (abi.BN_SPATIAL, abi.BN_PER_ACTIVATION):
        x = (rng.uniform(-1, 1, (3, 4, 5, 6)) * 2 + 0.3).astype(np.float32)
        dy = rng.uniform(-1, 1, x.shape).astype(np.float32)
        ns = 4 if mode == abi.BN_SPATIAL else 4 * 30
        g = rng.uniform(0.5, 1.5, ns).astype(np.float32)
        b = rng.uniform(-1, 1, ns).astype(np.float32)
        rm = rng.uniform(-1, 1, ns).astype(np.float32)
        rv = (1 + np.abs(rng.uniform(-1, 1, ns))).astype(np.float32)
        y, sm, si, rm2, rv2 = oracle.ref_bn_forward_train(mode, x, g, b, rm, rv)
        dx, dg, db = oracle.ref_bn_backward(mode, x, dy, g, b, sm, si)
        t = f"bn{mode}"
        for k, v in dict(x=x, dy=dy, g=g, b=b, rm=rm, rv=rv, y=y, sm=sm, si=si, rm2=rm2, rv2=rv2,
                         dx=dx, dg=dg, db=db).items():
            data[f"{t}_{k}"] = v
    # fused conv + bias + LeakyReLU (direct 1x1 row) and CBNA, both executors
    hf = ref.handle()
    for t, dims, fd, pad, stride, ops in (
            ("cba", (2, 4, 6, 6), (5, 4, 1, 1), 0, 1, ("bias", "leaky")),
            ("cbna", (2, 3, 9, 9), (4, 3, 3, 3), 1, 1, ("bias", "bn", "tanh"))):
        plan = ref.fusion_plan(dims)
        ref.check(plan.add_conv(fd, pad=pad, stride=stride))
        ref.check(plan.add_bias(fd[0]))
        if "bn" in ops:
            ref.check(plan.add_batchnorm(abi.BN_SPATIAL))
        ref.check(plan.add_activation(abi.LEAKY_RELU if "leaky" in ops else abi.TANH, 0.1))
        ref.check(plan.compile(hf))
        k = fd[0]
        args = dict(filter=rng.uniform(-1, 1, fd).astype(np.float32),
                    bias=rng.uniform(-1, 1, k).astype(np.float32),
                    gamma=rng.uniform(0.5, 1.5, k).astype(np.float32),
                    beta=rng.uniform(-1, 1, k).astype(np.float32),
                    mean=rng.uniform(-.5, .5, k).astype(np.float32),
                    var=(1 + rng.random(k)).astype(np.float32))
        plan.set_args(**args)
        x = rng.uniform(-1, 1, dims).astype(np.float32)
        data[f"{t}_x"] = x
        for kk, v in args.items():
            data[f"{t}_{kk}"] = v
        data[f"{t}_fused"] = plan.execute(hf, x)
        data[f"{t}_unfused"] = plan.execute(hf, x, unfused=True)
    np.savez_compressed(os.path.join(OUT, "reference_vectors.npz"), **data)
    print(f"wrote {len(data)} arrays to {OUT}/reference_vectors.npz")


if __name__ == "__main__":
    main()
