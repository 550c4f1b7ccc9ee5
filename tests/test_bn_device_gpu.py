"""Training batch-norm through the device C ABI (primkit_batchnorm_forward_train_device /
primkit_batchnorm_backward_device, bf16 NHWC) at sizes where the single-launch
persistent kernel (bn_coop.cu) spreads the rows over many CTAs and both grid
barriers matter: statistics, running statistics, y, dx, dgamma, dbeta against the
oracle restatement of primitives.cpp:61-152; bit-identical repeat runs
(deterministic reduction tree); the multi-kernel path (PK_BN_COOP=0 in a child
process) agrees within the bf16 tolerance."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi

from conftest import rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (n, c, h): ResNet-50-like channel counts / pitches, vpr = c/8 from 8 to 256
SHAPES = [(8, 64, 28), (16, 256, 14), (4, 2048, 7), (2, 40, 33)]


def _vp(t):
    return C.c_void_p(t.data_ptr())


def _run(lib, n, c, hh, relu, seed):
    rng = np.random.default_rng(seed)
    x = oracle.round_bf16(rng.uniform(-1, 1, (n, c, hh, hh)).astype(np.float32) * 2 + 0.3)
    dy = oracle.round_bf16(rng.uniform(-1, 1, (n, c, hh, hh)).astype(np.float32))
    g = rng.uniform(0.5, 1.5, c).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, c).astype(np.float32)
    rm, rv = rng.uniform(-0.2, 0.2, c).astype(np.float32), (1 + rng.random(c)).astype(np.float32)
    pitch = lib.channel_pitch(c)

    def nhwc(a):
        t = torch.from_numpy(a).permute(0, 2, 3, 1).contiguous()
        out = torch.zeros(t.shape[:-1] + (pitch,), dtype=torch.bfloat16)
        out[..., :c] = t.to(torch.bfloat16)
        return out.cuda()

    def nchw(t):
        return t[..., :c].float().permute(0, 3, 1, 2).contiguous().cpu().numpy()

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    xd, dyd = nhwc(x), nhwc(dy)
    yd, dxd = torch.zeros_like(xd), torch.zeros_like(xd)
    gd, bd, rmd, rvd = dev(g), dev(b), dev(rm), dev(rv)
    sm, si, dg, db = (torch.zeros(c, device="cuda") for _ in range(4))
    h = C.c_void_p()
    lib.check(lib.lib.primkit_handle_create_with_stream(C.c_void_p(0), 0, C.byref(h)))
    dims = (C.c_int64 * 4)(n, c, hh, hh)
    lib.check(lib.lib.primkit_batchnorm_forward_train_device(
        h, dims, abi.BF16, _vp(xd), _vp(gd), _vp(bd), _vp(rmd), _vp(rvd), C.c_float(1e-5),
        C.c_float(0.1), _vp(yd), _vp(sm), _vp(si), relu))
    lib.check(lib.lib.primkit_batchnorm_backward_device(
        h, dims, abi.BF16, _vp(xd), _vp(yd), _vp(dyd), _vp(gd), _vp(bd), _vp(sm), _vp(si),
        _vp(dxd), _vp(dg), _vp(db), relu))
    torch.cuda.synchronize()
    lib.lib.primkit_handle_destroy(h)
    host = lambda t: t.cpu().numpy()  # noqa: E731
    return dict(x=x, dy=dy, g=g, b=b, rm=rm, rv=rv, y=nchw(yd), dx=nchw(dxd), sm=host(sm),
                si=host(si), rm2=host(rmd), rv2=host(rvd), dg=host(dg), db=host(db))


@pytest.mark.parametrize("relu", [0, 1])
@pytest.mark.parametrize("shape", SHAPES)
def test_bn_device_matches_oracle(lib, shape, relu):
    n, c, hh = shape
    r = _run(lib, n, c, hh, relu, seed=n * 1000 + c + relu)
    oy, osm, osi, orm, orv = oracle.bn_forward_train(abi.BN_SPATIAL, r["x"], r["g"], r["b"], r["rm"], r["rv"],
                                                      bf16=True)
    np.testing.assert_allclose(r["sm"], osm, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(r["si"], osi, rtol=1e-5)
    np.testing.assert_allclose(r["rm2"], orm, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(r["rv2"], orv, rtol=1e-5)
    if relu:
        oy = np.maximum(oy, 0)
    assert rel_l2(r["y"], oy) <= 1e-2
    # ReLU backward: d = dy * (y > 0) on the stored BN output, then the reference BN backward
    dmask = r["dy"] * (r["y"] > 0) if relu else r["dy"]
    odx, odg, odb = oracle.bn_backward(abi.BN_SPATIAL, r["x"], dmask, r["g"], r["sm"], r["si"], bf16=True)
    assert rel_l2(r["dx"], odx) <= 1e-2
    assert rel_l2(r["dg"], odg) <= 1e-2 and rel_l2(r["db"], odb) <= 1e-2


def test_bn_device_deterministic(lib):
    a = _run(lib, 16, 256, 14, 1, seed=5)
    b = _run(lib, 16, 256, 14, 1, seed=5)
    for k in ("y", "dx", "sm", "si", "dg", "db"):
        assert np.array_equal(a[k], b[k]), k


def test_bn_device_multikernel_path_agrees(lib, tmp_path):
    """The legacy multi-kernel path (PK_BN_COOP=0) computes the same BN."""
    script = (
        "import sys, json, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from paper_1910_00078_b200.primkit import library\n"
        "import test_bn_device_gpu as t\n"
        "r = t._run(library(), 16, 256, 14, 1, seed=9)\n"
        "np.savez(%r, **{k: r[k] for k in ('y', 'dx', 'sm', 'si', 'dg', 'db')})\n"
    ) % (ROOT, os.path.join(ROOT, "tests"), str(tmp_path / "legacy.npz"))
    env = dict(os.environ, PK_BN_COOP="0")
    subprocess.check_call([sys.executable, "-c", script], env=env, cwd=ROOT)
    legacy = np.load(tmp_path / "legacy.npz")
    ours = _run(lib, 16, 256, 14, 1, seed=9)
    np.testing.assert_allclose(ours["sm"], legacy["sm"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(ours["si"], legacy["si"], rtol=1e-6)
    for k in ("y", "dx", "dg", "db"):
        assert rel_l2(ours[k], legacy[k]) <= 5e-3, k
