"""Convolution parity on the GPU through the C ABI: every (solver, direction,
element type) the registry admits, against the oracle restatement on the
same seeded inputs, plus the reference's counter and Find/tune contracts.

Tolerances (BASELINE.json north_star): f32 <= 1e-4 relative L2 (Winograd
<= 1e-3); bf16 <= 1e-2 relative L2 against the fp32 oracle on the same
bf16-rounded inputs. The reference's own max-rel metric is checked too."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import max_rel, rel_l2

pytestmark = pytest.mark.gpu

SHAPES = [
    dict(n=2, c=4, h=8, w=8, k=4, y=3, x=3, pad=1),
    dict(n=1, c=3, h=11, w=9, k=5, y=3, x=3, pad=1),
    dict(n=2, c=8, h=9, w=9, k=16, y=1, x=1),
    dict(n=1, c=6, h=12, w=10, k=4, y=5, x=3, pad_h=2, pad_w=1, stride=2),
    dict(n=2, c=4, h=10, w=10, k=6, y=3, x=3, pad=0, stride=1, dilation=2),
    dict(n=2, c=6, h=7, w=7, k=6, y=3, x=3, pad=1, groups=3),
    dict(n=1, c=16, h=14, w=14, k=32, y=3, x=3, pad=1),
    dict(n=2, c=64, h=8, w=8, k=64, y=3, x=3, pad=1),
    dict(n=1, c=32, h=9, w=9, k=48, y=1, x=1, stride=2),
    dict(n=1, c=3, h=20, w=20, k=8, y=7, x=7, pad=3, stride=2),
]


def _inputs(p, rng, bf16):
    sa, sb, _ = operand_shapes(oracle_lib(), p)
    a = rng.uniform(-1, 1, sa).astype(np.float32)
    b = rng.uniform(-1, 1, sb).astype(np.float32)
    if bf16:
        a, b = oracle.round_bf16(a), oracle.round_bf16(b)
    return a, b


def oracle_lib():
    from paper_1910_00078_b200.primkit import library
    return library()


def _oracle(p, a, b):
    if p.direction == abi.FORWARD:
        return oracle.conv_forward(p, a, b)
    if p.direction == abi.BACKWARD_DATA:
        return oracle.conv_backward_data(p, a, b)
    return oracle.conv_backward_weights(p, a, b)


def _cases():
    for i, s in enumerate(SHAPES):
        for et in (abi.F32, abi.BF16):
            for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
                yield pytest.param(i, et, d, id=f"s{i}-{'bf16' if et else 'f32'}-d{d}")


@pytest.mark.parametrize("si,et,direction", list(_cases()))
def test_every_applicable_solver(lib, si, et, direction):
    rng = np.random.default_rng(100 + si)
    p = problem(**SHAPES[si], direction=direction, etype=et)
    h = lib.handle()
    a, b = _inputs(p, rng, et == abi.BF16)
    want = _oracle(p, a, b)
    ran = 0
    for s in h.solver_names():
        if not h.is_applicable(s, p):
            continue
        got = h.conv_run(p, s, a, b)
        tol = (1e-2 if et == abi.BF16 else (1e-3 if s in ("Winograd", "FFT") else 1e-4))
        err = rel_l2(got, want)
        assert err <= tol, f"{s} {h.last_kernel()} rel-L2 {err:.3e}"
        if et == abi.BF16:
            # outputs are bf16 values (round on store)
            assert np.array_equal(oracle.round_bf16(got), got)
        else:
            assert max_rel(got, want) <= (1e-3 if s in ("Winograd", "FFT") else 1e-4)
        ran += 1
    assert ran >= 2


def test_transpose_mode(lib):
    rng = np.random.default_rng(5)
    h = lib.handle()
    for shp in (dict(n=1, c=4, h=7, w=7, k=2, y=3, x=3, pad=1, stride=2),
                dict(n=2, c=6, h=5, w=6, k=4, y=2, x=3, pad=0, stride=1, groups=2)):
        p = problem(**shp, mode=abi.TRANSPOSE)
        a, b = _inputs(p, rng, False)
        want = oracle.conv_ref_f64(*_transpose_as_conv(p, a, b))
        for s in ("Direct", "Im2colGemm"):
            got = h.conv_run(p, s, a, b)
            assert rel_l2(got, want) <= 1e-4, s


@pytest.mark.parametrize("et", [abi.F32, abi.BF16])
def test_transpose_mode_tiled(lib, et):
    """Transpose-mode forward on the Direct solver runs the register-tiled
    backward-data kernel with the roles of input and output swapped."""
    rng = np.random.default_rng(6)
    h = lib.handle()
    for shp in (dict(n=2, c=32, h=9, w=8, k=24, y=3, x=3, pad=1, stride=2),
                dict(n=1, c=16, h=6, w=7, k=72, y=4, x=4, pad=1, stride=2),
                dict(n=2, c=8, h=5, w=5, k=8, y=3, x=3, pad=0, stride=1),
                dict(n=1, c=70, h=4, w=4, k=3, y=3, x=3, pad=2, stride=3)):
        p = problem(**shp, mode=abi.TRANSPOSE, etype=et)
        a, b = _inputs(p, rng, et == abi.BF16)
        want = oracle.conv_ref_f64(*_transpose_as_conv(p, a, b))
        got = h.conv_run(p, "Direct", a, b)
        assert h.last_kernel() == "direct_simt_tiled_transpose", h.last_kernel()
        assert rel_l2(got, want) <= (1e-2 if et == abi.BF16 else 1e-4), shp


def _transpose_as_conv(p, x, w):
    """Transpose conv == stride-1 conv of the zero-upsampled input with the
    flipped, channel-swapped filter (independent formulation)."""
    st = p.stride_h
    cg, kg = p.c // p.groups, p.k // p.groups
    up_h, up_w = (p.h - 1) * st + 1, (p.w - 1) * p.stride_w + 1
    xu = np.zeros((p.n, p.c, up_h, up_w), np.float32)
    xu[:, :, ::st, ::p.stride_w] = x
    wf = np.zeros((p.k, cg, p.y, p.x), np.float32)
    for g in range(p.groups):
        for c in range(cg):
            for kk in range(kg):
                wf[g * kg + kk, c] = w[g * cg + c, kk, ::-1, ::-1]
    q = problem(n=p.n, c=p.c, h=up_h, w=up_w, k=p.k, y=p.y, x=p.x, pad_h=p.y - 1 - p.pad_h,
                pad_w=p.x - 1 - p.pad_w, groups=p.groups)
    return q, xu, wf


def test_counters_match_reference(lib, ref):
    rng = np.random.default_rng(9)
    h, hr = lib.handle(), ref.handle()
    for shp in SHAPES[:6]:
        for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
            p = problem(**shp, direction=d)
            a, b = _inputs(p, rng, False)
            for s in h.solver_names():
                if not h.is_applicable(s, p):
                    continue
                h.reset_counters()
                hr.reset_counters()
                h.conv_run(p, s, a, b)
                hr.conv_run(p, s, a, b)
                assert h.counters() == hr.counters(), (s, d, shp)


def test_winograd_multiplies(lib):
    # acceptance.cpp:162-186: 16 muls per (tile, channel, k) vs 36 direct
    h = lib.handle()
    p = problem(n=1, c=1, h=4, w=4, k=1, y=3, x=3)
    x = np.ones((1, 1, 4, 4), np.float32)
    w = np.ones((1, 1, 3, 3), np.float32)
    h.conv_run(p, "Winograd", x, w)
    assert h.counters()[1] == 16
    h.reset_counters()
    h.conv_run(p, "Direct", x, w)
    assert h.counters()[1] == 36


def test_known_answers(lib):
    h = lib.handle()
    # test_conv.cpp:127-136: 3x3 iota input, 2x2 ones filter -> [[8,12],[20,24]]
    x = np.arange(0, 9, dtype=np.float32).reshape(1, 1, 3, 3)
    w = np.ones((1, 1, 2, 2), np.float32)
    p = problem(n=1, c=1, h=3, w=3, k=1, y=2, x=2)
    for s in ("Direct", "Im2colGemm", "FFT", "ImplicitGemm"):
        np.testing.assert_allclose(h.conv_run(p, s, x, w).ravel(), [8, 12, 20, 24], rtol=1e-6)
    # test_capi.cpp:168-194: 1x1 filter 2*I scales the input by two
    rng = np.random.default_rng(112)
    p = problem(n=1, c=4, h=8, w=8, k=4)
    a = rng.uniform(-1, 1, (1, 4, 8, 8)).astype(np.float32)
    b = (2.0 * np.eye(4, dtype=np.float32)).reshape(4, 4, 1, 1)
    for s in ("Direct", None):
        np.testing.assert_allclose(h.conv_run(p, s, a, b, 1 << 22), 2 * a, rtol=1e-6)


def test_implicit_gemm_bit_identical_across_tiles(lib):
    # test_conv.cpp:211-235: results do not depend on the tile configuration
    rng = np.random.default_rng(3)
    for et in (abi.F32, abi.BF16):
        p = problem(n=2, c=16, h=12, w=12, k=32, y=3, x=3, pad=1, etype=et)
        a, b = _inputs(p, rng, et == abi.BF16)
        h = lib.handle()
        base = h.conv_run(p, "ImplicitGemm", a, b)
        import tempfile
        for tm, tn, tk in ((2, 1, 1), (4, 2, 2), (8, 4, 4)):
            with tempfile.NamedTemporaryFile("w", suffix=".db", delete=False) as f:
                f.write(f"{lib.problem_key(p)}=ImplicitGemm:{tm},{tn},{tk}\n")
            h2 = lib.handle()
            h2.perfdb_load(f.name)
            assert np.array_equal(h2.conv_run(p, "ImplicitGemm", a, b), base)


def test_find_sorted_and_workspace_filtered(lib):
    h = lib.handle()
    h.use_fake_clock()
    p = problem(n=1, c=4, h=8, w=8, k=4, y=3, x=3, pad=1)
    rng = np.random.default_rng(111)
    a = rng.uniform(-1, 1, (1, 4, 8, 8)).astype(np.float32)
    b = rng.uniform(-1, 1, (4, 4, 3, 3)).astype(np.float32)
    rows, found = h.find(p, a, b, 1 << 22, 8)
    assert found == 5 and len(rows) == 5
    assert all(rows[i].time_ms <= rows[i + 1].time_ms for i in range(4))
    rows, found = h.find(p, a, b, 0, 8)
    assert all(r.workspace_bytes == 0 for r in rows)
    # real device timing
    h2 = lib.handle()
    rows, found = h2.find(p, a, b, 1 << 22, 8)
    assert found == 5 and all(r.time_ms > 0 for r in rows)
    assert [r.time_ms for r in rows] == sorted(r.time_ms for r in rows)


def test_tune_writes_perfdb(lib, tmp_path):
    h = lib.handle()
    h.use_fake_clock()
    p = problem(n=1, c=4, h=6, w=6, k=4, y=3, x=3, pad=1)
    assert h.tune(p, "ImplicitGemm", 4) >= 1
    path = tmp_path / "db.txt"
    h.perfdb_save(str(path))
    text = path.read_text()
    assert text.startswith("1-4-6-6-4-3-3-1-1-1-1-1-1-1-F-C-f32=ImplicitGemm:")
    # full device-timed tune over the whole grid
    h2 = lib.handle()
    # grid {1,2,4,8}^2 x {1,2,4} filtered by k=4, 36 pixels, c=4 divisibility: 3*3*3
    assert h2.tune(p, "ImplicitGemm", 0, exhaustive=True) == 27


def test_bf16_large_tensor_core_paths(lib):
    """ResNet-50-shaped layers at reduced N through the tcgen05 kernels."""
    rng = np.random.default_rng(21)
    h = lib.handle()
    for shp in (dict(n=2, c=64, h=56, w=56, k=64, y=3, x=3, pad=1),
                dict(n=2, c=256, h=14, w=14, k=256, y=3, x=3, pad=1),
                dict(n=2, c=64, h=56, w=56, k=256, y=1, x=1),
                dict(n=2, c=128, h=28, w=28, k=128, y=3, x=3, pad=1, stride=2),
                dict(n=3, c=128, h=28, w=28, k=128, y=3, x=3, pad=1),   # 256-px rectangles (MT=2)
                dict(n=2, c=128, h=15, w=13, k=64, y=3, x=3, pad=1),    # MT=2, ragged, BN=64
                dict(n=2, c=64, h=56, w=56, k=128, y=1, x=1),           # resident-filter 1x1
                dict(n=2, c=512, h=7, w=7, k=128, y=1, x=1),            # resident 128 KB slice
                dict(n=8, c=512, h=56, w=56, k=256, y=1, x=1),          # CTA-pair GEMM (fwd)
                dict(n=8, c=256, h=56, w=56, k=512, y=1, x=1),          # CTA-pair GEMM (dgrad)
                dict(n=2, c=512, h=14, w=14, k=1024, y=1, x=1, stride=2),
                dict(n=2, c=3, h=32, w=32, k=64, y=7, x=7, pad=3, stride=2),
                dict(n=1, c=256, h=13, w=13, k=512, y=1, x=1, stride=2)):
        for d, s, kern in ((abi.FORWARD, "ImplicitGemm", "igemm_tc_fwd"),
                           (abi.BACKWARD_DATA, "Im2colGemm", "igemm_tc_dgrad"),
                           (abi.BACKWARD_WEIGHTS, "Im2colGemm", "igemm_tc_wgrad")):
            p = problem(**shp, direction=d, etype=abi.BF16)
            a, b = _inputs(p, rng, True)
            got = h.conv_run(p, s, a, b)
            # narrow-channel stems pack (r,s,c) densely before the tcgen05 GEMMs
            assert h.last_kernel() == kern or (shp["c"] % 64 and h.last_kernel().startswith("stem"))
            err = rel_l2(got, _oracle(p, a, b))
            assert err <= 1e-2, (shp, d, err)
