"""Pin the oracle before trusting it (CPU suite).

1. The reference's own known-answer tests (test_tensor.cpp:12-48,
   test_conv.cpp:127-136, acceptance.cpp:162-186).
2. The golden vectors produced by the unmodified reference
   (tests/golden/reference_vectors.npz, made by tests/golden/make_golden.py).
3. Live call-by-call comparison with the reference library (oracle/_ref) on
   seeded random problems, when it is built here.
"""
import os

import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import max_rel

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


def test_round_bf16_known_answers():
    r = oracle.restated()
    f = r.oc_round_bf16
    assert f(1.0) == 1.0 and f(2.0) == 2.0 and f(-3.5) == -3.5
    assert f(1.00390625) == 1.0            # tie to even (kept lsb 0)
    assert f(1.01171875) == 1.015625       # tie rounds up (kept lsb 1)
    assert np.isinf(f(float("inf"))) and f(float("-inf")) < 0 and np.isnan(f(float("nan")))
    assert np.signbit(f(-0.0))


def test_round_bf16_vectorised_idempotent():
    rng = np.random.default_rng(7)
    x = rng.uniform(-1e6, 1e6, 10000).astype(np.float32)
    r = oracle.round_bf16(x)
    assert np.array_equal(oracle.round_bf16(r), r)
    assert np.all((r.view(np.uint32) & 0xFFFF) == 0)
    lib = oracle.restated()
    assert all(lib.oc_round_bf16(float(v)) == float(w) for v, w in zip(x[:500], r[:500]))


def test_direct_hand_example():
    x = np.arange(9, dtype=np.float32).reshape(1, 1, 3, 3)
    w = np.ones((1, 1, 2, 2), np.float32)
    y = oracle.conv_forward(problem(n=1, c=1, h=3, w=3, k=1, y=2, x=2), x, w)
    assert y.ravel().tolist() == [8.0, 12.0, 20.0, 24.0]


def test_winograd_matches_direct():
    rng = np.random.default_rng(23)
    p = problem(n=2, c=8, h=16, w=16, k=4, y=3, x=3, pad=1)
    x = rng.uniform(-1, 1, (2, 8, 16, 16)).astype(np.float32)
    w = rng.uniform(-1, 1, (4, 8, 3, 3)).astype(np.float32)
    assert max_rel(oracle.winograd_f23(p, x, w), oracle.conv_forward(p, x, w)) <= 1e-4


def test_direct_matches_independent_f64():
    rng = np.random.default_rng(5)
    for shp in (dict(n=2, c=6, h=9, w=7, k=4, y=3, x=2, pad_h=1, pad_w=0, stride=2, dilation=1,
                     groups=2),
                dict(n=1, c=3, h=11, w=11, k=5, y=3, x=3, pad=2, dilation=2)):
        p = problem(**shp)
        sa, sb, _ = operand_shapes(_lib(), p)
        x = rng.uniform(-1, 1, sa).astype(np.float32)
        w = rng.uniform(-1, 1, sb).astype(np.float32)
        assert max_rel(oracle.conv_forward(p, x, w), oracle.conv_ref_f64(p, x, w)) <= 1e-5


def test_backward_is_adjoint_of_forward():
    # <conv(x, w), dy> == <x, conv_bd(dy, w)> == <w, conv_bw(dy, x)> (test_conv.cpp:387-413)
    rng = np.random.default_rng(11)
    p = problem(n=2, c=4, h=8, w=7, k=3, y=3, x=3, pad=1, stride=2)
    x = rng.uniform(-1, 1, (2, 4, 8, 7))
    w = rng.uniform(-1, 1, (3, 4, 3, 3))
    y = oracle.conv_forward(p, x, w)
    dy = rng.uniform(-1, 1, y.shape)
    lhs = float(np.sum(y.astype(np.float64) * dy))
    assert abs(lhs - float(np.sum(oracle.conv_backward_data(p, dy, w) * x))) <= 1e-4 * abs(lhs) + 1e-4
    assert abs(lhs - float(np.sum(oracle.conv_backward_weights(p, dy, x) * w))) <= 1e-4 * abs(lhs) + 1e-4


def _lib():
    from paper_1910_00078_b200.primkit import library
    return library()


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _golden_cases():
    # the case table lives next to the fixtures, in the generator script
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "make_golden", os.path.join(os.path.dirname(GOLDEN), "make_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.CONV_CASES


@pytest.mark.parametrize("case", [c[0] for c in _golden_cases()])
@pytest.mark.parametrize("et", [abi.F32, abi.BF16])
def test_oracle_matches_reference_golden(golden, case, et):
    name, shp, d = next(c for c in _golden_cases() if c[0] == case)
    p = problem(**shp, direction=d, etype=et)
    tag = f"{name}_{'bf16' if et else 'f32'}"
    a, b = golden[tag + "_a"], golden[tag + "_b"]
    bf = et == abi.BF16
    got = {abi.FORWARD: oracle.conv_forward, abi.BACKWARD_DATA: oracle.conv_backward_data,
           abi.BACKWARD_WEIGHTS: oracle.conv_backward_weights}[d](p, a, b, bf16=bf)
    # same loop order and f32 arithmetic as the reference: bit-identical
    assert np.array_equal(got, golden[tag + "_direct"])
    if tag + "_winograd" in golden.files:
        assert np.array_equal(oracle.winograd_f23(p, a, b, bf16=bf), golden[tag + "_winograd"])


@pytest.mark.parametrize("mode", [abi.BN_SPATIAL, abi.BN_PER_ACTIVATION])
def test_oracle_bn_matches_reference_golden(golden, mode):
    t = f"bn{mode}"
    G = {k: golden[f"{t}_{k}"] for k in ("x", "dy", "g", "b", "rm", "rv", "y", "sm", "si", "rm2",
                                          "rv2", "dx", "dg", "db")}
    y, sm, si, rm, rv = oracle.bn_forward_train(mode, G["x"], G["g"], G["b"], G["rm"], G["rv"])
    for got, want in ((y, "y"), (sm, "sm"), (si, "si"), (rm, "rm2"), (rv, "rv2")):
        assert np.array_equal(got, G[want]), want
    dx, dg, db = oracle.bn_backward(mode, G["x"], G["dy"], G["g"], G["sm"], G["si"])
    assert max_rel(dx, G["dx"]) <= 1e-6 and max_rel(dg, G["dg"]) <= 1e-6
    assert max_rel(db, G["db"]) <= 1e-6


def test_oracle_fused_epilogue_matches_reference_golden(golden):
    r = oracle.restated()
    for t, pad, act, has_bn in (("cba", 0, abi.LEAKY_RELU, False), ("cbna", 1, abi.TANH, True)):
        x, w = golden[f"{t}_x"], golden[f"{t}_filter"]
        p = problem(n=x.shape[0], c=x.shape[1], h=x.shape[2], w=x.shape[3], k=w.shape[0],
                    y=w.shape[2], x=w.shape[3], pad=pad)
        conv = oracle.conv_forward(p, x, w)
        out = np.empty_like(conv)
        for k in range(conv.shape[1]):
            for idx in np.ndindex(conv.shape[0], conv.shape[2], conv.shape[3]):
                n, i, j = idx
                out[n, k, i, j] = r.oc_fused_epilogue(
                    float(conv[n, k, i, j]), 1, float(golden[f"{t}_bias"][k]), int(has_bn),
                    float(golden[f"{t}_mean"][k]), float(golden[f"{t}_var"][k]),
                    float(golden[f"{t}_gamma"][k]), float(golden[f"{t}_beta"][k]), 1e-5, act, 0.1)
        assert max_rel(out, golden[f"{t}_fused"]) <= 1e-6
        assert max_rel(golden[f"{t}_fused"], golden[f"{t}_unfused"]) <= 1e-5


def test_oracle_matches_live_reference(ref):
    """Random problems, every direction, through the reference's C ABI."""
    h = ref.handle()
    rng = np.random.default_rng(99)
    for _ in range(40):
        shp = dict(n=int(rng.integers(1, 3)), c=int(rng.integers(1, 6)), h=int(rng.integers(3, 9)),
                   w=int(rng.integers(3, 9)), k=int(rng.integers(1, 6)), y=int(rng.integers(1, 4)),
                   x=int(rng.integers(1, 4)), pad=int(rng.integers(0, 2)),
                   stride=int(rng.integers(1, 3)), dilation=int(rng.integers(1, 3)))
        for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
            p = problem(**shp, direction=d)
            try:
                sa, sb, _ = operand_shapes(ref, p)
            except Exception:
                break  # invalid geometry
            a = rng.uniform(-1, 1, sa).astype(np.float32)
            b = rng.uniform(-1, 1, sb).astype(np.float32)
            want = h.conv_run(p, "Direct", a, b)
            got = {abi.FORWARD: oracle.conv_forward, abi.BACKWARD_DATA: oracle.conv_backward_data,
                   abi.BACKWARD_WEIGHTS: oracle.conv_backward_weights}[d](p, a, b)
            assert np.array_equal(got, want), (shp, d)


def _to_dev(a, pitch):
    """NCHW f32 -> NHWC with channel pitch (zero pad lanes)."""
    n, c, h, w = a.shape
    out = np.zeros((n, h, w, pitch), np.float32)
    out[..., :c] = a.transpose(0, 2, 3, 1)
    return out


def _bits(a):
    return np.ascontiguousarray((oracle.round_bf16(a).view(np.uint32) >> 16).astype(np.uint16))


@pytest.mark.parametrize("cfg", [
    dict(n=2, c=5, h=9, w=7, k=6, y=3, x=3, pad=1),
    dict(n=2, c=16, h=11, w=11, k=8, y=3, x=3, pad=1, stride=2),
    dict(n=1, c=3, h=15, w=15, k=8, y=7, x=7, pad=3, stride=2),
    dict(n=2, c=8, h=8, w=8, k=16, y=1, x=1, stride=2),
    dict(n=1, c=8, h=9, w=9, k=8, y=3, x=3, pad=2, dilation=2),
])
@pytest.mark.parametrize("bf16", [False, True])
def test_sampled_formulas_match_full_oracle(cfg, bf16):
    """The device-layout sampled formulas (used for full-size GPU parity) give
    the full restated oracle's values at every coordinate."""
    from paper_1910_00078_b200.primkit import problem
    rng = np.random.default_rng(5)
    p = problem(**cfg)
    oh, ow = oracle.out_hw(p)
    x = oracle.round_bf16(rng.uniform(-1, 1, (p.n, p.c, p.h, p.w)).astype(np.float32))
    w = oracle.round_bf16(rng.uniform(-1, 1, (p.k, p.c, p.y, p.x)).astype(np.float32))
    dy = oracle.round_bf16(rng.uniform(-1, 1, (p.n, p.k, oh, ow)).astype(np.float32))
    pit = lambda c: (c + 7) // 8 * 8  # noqa: E731
    xd, dyd = _to_dev(x, pit(p.c)), _to_dev(dy, pit(p.k))
    wd = _to_dev(w, pit(p.c))  # [K][R][S][pitch C]
    conv = (lambda a: _bits(a)) if bf16 else (lambda a: np.ascontiguousarray(a, np.float32))
    xd, dyd, wd = conv(xd), conv(dyd), conv(wd)

    y = oracle.conv_ref_f64(p, x, w)
    idx = np.array([(n, k, i, j) for n in range(p.n) for k in range(p.k) for i in range(oh)
                    for j in range(ow)], np.int64)
    got = oracle.sample_forward(p, xd, wd, idx, bf16)
    np.testing.assert_allclose(got, y[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]], rtol=1e-9, atol=1e-9)

    dx = oracle.conv_backward_data(p, dy, w).astype(np.float64)
    idx = np.array([(n, c, i, j) for n in range(p.n) for c in range(p.c) for i in range(p.h)
                    for j in range(p.w)], np.int64)
    got = oracle.sample_backward_data(p, dyd, wd, idx, bf16)
    np.testing.assert_allclose(got, dx[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]], rtol=1e-5, atol=1e-5)

    dw = oracle.conv_backward_weights(p, dy, x).astype(np.float64)
    taps = np.array([(r, s, c) for r in range(p.y) for s in range(p.x) for c in range(p.c)], np.int64)
    ks = np.arange(p.k)
    got = oracle.sample_backward_weights(p, dyd, xd, ks, taps, bf16)
    want = dw[ks][:, taps[:, 2], taps[:, 0], taps[:, 1]]
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-4)


POOL_CASES = [
    ((2, 3, 7, 7), (3, 3), (1, 1), (2, 2)),      # ResNet stem max-pool shape, padded
    ((1, 2, 6, 5), (2, 2), (0, 0), (2, 2)),
    ((2, 2, 5, 5), (3, 2), (1, 0), (1, 2)),       # overlapping windows
    ((1, 1, 3, 3), (5, 5), (2, 2), (3, 3)),       # windows larger than the image
    ((1, 4, 7, 7), (7, 7), (0, 0), (1, 1)),       # global average pool
]


@pytest.mark.parametrize("case", POOL_CASES)
@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("bf16", [False, True])
def test_pooling_restatement_matches_reference(ref, case, kind, bf16):
    dims, win, pad, stride = case
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, dims).astype(np.float32)
    x[0, 0, 0, :2] = 0.5  # ties: the first maximum wins
    if bf16:
        x = oracle.round_bf16(x)
    y, idx = oracle.pool_forward(kind, x, win, pad, stride, bf16)
    yr, idxr = oracle.ref_pool_forward(kind, x, win, pad, stride, bf16)
    assert np.array_equal(y, yr) and np.array_equal(idx, idxr)
    dy = rng.uniform(-1, 1, y.shape).astype(np.float32)
    if bf16:
        dy = oracle.round_bf16(dy)
    dx = oracle.pool_backward(kind, dims, dy, idx, win, pad, stride, bf16)
    dxr = oracle.ref_pool_backward(kind, dims, dy, idxr, win, pad, stride, bf16)
    assert np.array_equal(dx, dxr)


@pytest.mark.parametrize("shape,axis", [((4, 10), 1), ((2, 5, 3, 3), 1), ((3, 7), 0), ((2, 3, 4), 2)])
@pytest.mark.parametrize("bf16", [False, True])
def test_softmax_restatement_matches_reference(ref, shape, axis, bf16):
    rng = np.random.default_rng(9)
    x = rng.uniform(-4, 4, shape).astype(np.float32)
    if bf16:
        x = oracle.round_bf16(x)
    y = oracle.softmax_forward(x, axis, bf16)
    assert np.array_equal(y, oracle.ref_softmax_forward(x, axis, bf16))
    dy = rng.uniform(-1, 1, shape).astype(np.float32)
    if bf16:
        dy = oracle.round_bf16(dy)
    assert np.array_equal(oracle.softmax_backward(y, dy, axis, bf16),
                          oracle.ref_softmax_backward(y, dy, axis, bf16))
