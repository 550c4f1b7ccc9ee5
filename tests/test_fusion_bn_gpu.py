"""Fusion plans, batch-norm and activation on the GPU against the oracle and
the reference's fused==unfused contracts (test_fusion.cpp:276-478,
test_primitives.cpp)."""
import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import problem

from conftest import max_rel, rel_l2

pytestmark = pytest.mark.gpu


def _args(rng, k, c, f, mode, hw, bf16):
    w = rng.uniform(-1, 1, (k, c, f, f)).astype(np.float32)
    if bf16:
        w = oracle.round_bf16(w)
    ns = k if mode == abi.BN_SPATIAL else k * hw
    return dict(filter=w, bias=rng.uniform(-1, 1, k).astype(np.float32),
                gamma=rng.uniform(0.5, 1.5, ns).astype(np.float32),
                beta=rng.uniform(-1, 1, ns).astype(np.float32),
                mean=rng.uniform(-0.5, 0.5, ns).astype(np.float32),
                var=(1 + np.abs(rng.uniform(-1, 1, ns))).astype(np.float32))


def _oracle_fused(x, a, conv_p, ops, bn_mode, alpha, eps=1e-5):
    y = oracle.conv_ref_f64(conv_p, x, a["filter"])
    k = y.shape[1]
    for op in ops:
        if op == "bias":
            y = y + a["bias"][None, :, None, None]
        elif op == "bn":
            shape = (1, k, 1, 1) if bn_mode == abi.BN_SPATIAL else (1, k, y.shape[2], y.shape[3])
            g, b, m, v = (a[n].reshape(shape) for n in ("gamma", "beta", "mean", "var"))
            y = (y - m) / np.sqrt(v + eps) * g + b
        else:
            kind = op[1]
            if kind == abi.RELU:
                y = np.maximum(y, 0)
            elif kind == abi.LEAKY_RELU:
                y = np.where(y > 0, y, alpha * y)
            elif kind == abi.SIGMOID:
                y = 1 / (1 + np.exp(-y))
            else:
                y = np.tanh(y)
    return y


CASES = [
    # dims, etype, filter, pad, stride, algo, ops, bn_mode
    ((2, 4, 6, 6), abi.F32, (5, 4, 1, 1), 0, 1, "Direct", ["bias", ("act", abi.SIGMOID)], 1),
    ((2, 3, 9, 9), abi.F32, (4, 3, 3, 3), 1, 1, "Direct", ["bias", "bn", ("act", abi.TANH)], 1),
    ((2, 3, 9, 9), abi.F32, (4, 3, 3, 3), 1, 1, "Direct", ["bias", "bn", ("act", abi.TANH)], 0),
    ((1, 18, 12, 12), abi.F32, (6, 18, 3, 3), 1, 1, "Winograd", ["bias", ("act", abi.LEAKY_RELU)], 1),
    ((1, 20, 12, 12), abi.F32, (6, 20, 5, 5), 2, 2, "Winograd", ["bias", ("act", abi.RELU)], 1),
    ((2, 64, 8, 8), abi.BF16, (64, 64, 1, 1), 0, 1, "Direct", ["bias", ("act", abi.RELU)], 1),
    ((2, 64, 14, 14), abi.BF16, (256, 64, 1, 1), 0, 1, "Direct", ["bias", ("act", abi.RELU)], 1),
    ((2, 16, 9, 9), abi.BF16, (32, 16, 3, 3), 1, 2, "Direct", ["bias", "bn", ("act", abi.RELU)], 1),
    ((2, 8, 9, 9), abi.BF16, (16, 8, 5, 5), 2, 1, "Direct", ["bias", "bn", ("act", abi.SIGMOID)], 0),
]


def _plan(lib, h, case, rng):
    dims, et, fd, pad, stride, algo, ops, mode = case
    plan = lib.fusion_plan(dims, et)
    lib.check(plan.add_conv(fd, pad=pad, stride=stride, algo=algo))
    for op in ops:
        if op == "bias":
            lib.check(plan.add_bias(fd[0]))
        elif op == "bn":
            lib.check(plan.add_batchnorm(mode))
        else:
            lib.check(plan.add_activation(op[1], 0.2))
    lib.check(plan.compile(h))
    od = plan.output_dims()
    a = _args(rng, fd[0], fd[1], fd[2], mode, od[2] * od[3], et == abi.BF16)
    plan.set_args(**a)
    return plan, a


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_fused_equals_unfused_and_oracle(lib, ci):
    case = CASES[ci]
    dims, et, fd, pad, stride, algo, ops, mode = case
    rng = np.random.default_rng(200 + ci)
    h = lib.handle()
    plan, a = _plan(lib, h, case, rng)
    x = rng.uniform(-1, 1, dims).astype(np.float32)
    if et == abi.BF16:
        x = oracle.round_bf16(x)
    h.reset_counters()
    fused = plan.execute(h, x)
    assert h.counters()[2] == 1  # one buffer round trip
    h.reset_counters()
    unfused = plan.execute(h, x, unfused=True)
    assert h.counters()[2] == 1 + len(ops)
    tol = 2e-2 if et == abi.BF16 else 1e-5
    assert max_rel(fused, unfused) <= tol
    conv_p = problem(n=dims[0], c=dims[1], h=dims[2], w=dims[3], k=fd[0], y=fd[2], x=fd[3],
                     pad=pad, stride=stride)
    want = _oracle_fused(x, a, conv_p, ops, mode, 0.2)
    assert rel_l2(fused, want) <= (1e-2 if et == abi.BF16 else 1e-4)


def test_fused_matches_reference_library(lib, ref):
    rng = np.random.default_rng(300)
    for case in CASES[:5]:
        h, hr = lib.handle(), ref.handle()
        plan, a = _plan(lib, h, case, rng)
        rplan, _ = _plan(ref, hr, case, np.random.default_rng(0))
        rplan.set_args(**a)
        x = rng.uniform(-1, 1, case[0]).astype(np.float32)
        for unf in (False, True):
            h.reset_counters()
            hr.reset_counters()
            got = plan.execute(h, x, unfused=unf)
            want = rplan.execute(hr, x, unfused=unf)
            assert max_rel(got, want) <= 1e-5
            assert h.counters() == hr.counters()


def test_neutral_epilogue_bit_equal_to_plain_conv(lib):
    # test_fusion.cpp:361-385
    rng = np.random.default_rng(105)
    h = lib.handle()
    plan = lib.fusion_plan((1, 4, 5, 5))
    lib.check(plan.add_conv((4, 4, 1, 1)))
    lib.check(plan.add_bias(4))
    lib.check(plan.add_activation(abi.LEAKY_RELU, 1.0))
    lib.check(plan.compile(h))
    w = rng.uniform(-1, 1, (4, 4, 1, 1)).astype(np.float32)
    plan.set_args(filter=w, bias=np.zeros(4, np.float32))
    x = rng.uniform(-1, 1, (1, 4, 5, 5)).astype(np.float32)
    fused = plan.execute(h, x)
    plain = h.conv_run(problem(n=1, c=4, h=5, w=5, k=4), "Direct", x, w)
    assert np.array_equal(fused, plain)


def test_norm_activation(lib):
    rng = np.random.default_rng(104)
    h = lib.handle()
    plan = lib.fusion_plan((2, 5, 4, 4))
    lib.check(plan.add_batchnorm(abi.BN_PER_ACTIVATION))
    lib.check(plan.add_activation(abi.RELU))
    lib.check(plan.compile(h))
    ns = 5 * 16
    g, b = rng.uniform(0.5, 1.5, ns).astype(np.float32), rng.uniform(-1, 1, ns).astype(np.float32)
    m, v = rng.uniform(-.5, .5, ns).astype(np.float32), (1 + rng.random(ns)).astype(np.float32)
    plan.set_args(gamma=g, beta=b, mean=m, var=v)
    x = rng.uniform(-1, 1, (2, 5, 4, 4)).astype(np.float32)
    h.reset_counters()
    fused = plan.execute(h, x)
    assert h.counters()[2] == 1
    h.reset_counters()
    unfused = plan.execute(h, x, unfused=True)
    assert h.counters()[2] == 2
    assert max_rel(fused, unfused) <= 1e-5
    want = np.maximum(oracle.bn_forward_infer(0, x, g, b, m, v), 0)
    assert max_rel(fused, want) <= 1e-5


@pytest.mark.parametrize("mode", [abi.BN_SPATIAL, abi.BN_PER_ACTIVATION])
@pytest.mark.parametrize("et", [abi.F32, abi.BF16])
def test_batchnorm_train_and_backward(lib, mode, et):
    rng = np.random.default_rng(40 + mode + 2 * et)
    h = lib.handle()
    shape = (4, 6, 5, 7)
    x = rng.uniform(-1, 1, shape).astype(np.float32) * 3 + 0.5
    dy = rng.uniform(-1, 1, shape).astype(np.float32)
    if et == abi.BF16:
        x, dy = oracle.round_bf16(x), oracle.round_bf16(dy)
    ns = 6 if mode == abi.BN_SPATIAL else 6 * 35
    g = rng.uniform(0.5, 1.5, ns).astype(np.float32)
    b = rng.uniform(-1, 1, ns).astype(np.float32)
    rm, rv = rng.uniform(-1, 1, ns).astype(np.float32), (1 + rng.random(ns)).astype(np.float32)
    y, sm, si, rm2, rv2 = h.bn_forward_train(mode, x, g, b, rm, rv, etype=et)
    oy, osm, osi, orm, orv = oracle.bn_forward_train(mode, x, g, b, rm, rv, bf16=et == abi.BF16)
    tol = 1e-2 if et == abi.BF16 else 1e-4
    assert rel_l2(y, oy) <= tol
    np.testing.assert_allclose(sm, osm, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(si, osi, rtol=1e-5)
    np.testing.assert_allclose(rm2, orm, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(rv2, orv, rtol=1e-5)
    dx, dg, db = h.bn_backward(mode, x, dy, g, sm, si, etype=et)
    odx, odg, odb = oracle.bn_backward(mode, x, dy, g, sm, si, bf16=et == abi.BF16)
    assert rel_l2(dx, odx) <= tol
    assert rel_l2(dg, odg) <= tol and rel_l2(db, odb) <= tol
    infer = h.bn_forward_infer(mode, x, g, b, rm, rv, etype=et)
    assert rel_l2(infer, oracle.bn_forward_infer(mode, x, g, b, rm, rv,
                                                 bf16=et == abi.BF16)) <= tol


def test_batchnorm_matches_reference_library(lib, ref):
    rng = np.random.default_rng(77)
    h = lib.handle()
    for mode in (abi.BN_SPATIAL, abi.BN_PER_ACTIVATION):
        shape = (3, 4, 6, 5)
        x = rng.uniform(-2, 2, shape).astype(np.float32)
        dy = rng.uniform(-1, 1, shape).astype(np.float32)
        ns = 4 if mode == abi.BN_SPATIAL else 4 * 30
        g, b = rng.uniform(0.5, 1.5, ns).astype(np.float32), rng.uniform(-1, 1, ns).astype(np.float32)
        rm, rv = np.zeros(ns, np.float32), np.ones(ns, np.float32)
        y, sm, si, _, _ = h.bn_forward_train(mode, x, g, b, rm, rv)
        ry, rsm, rsi, _, _ = oracle.ref_bn_forward_train(mode, x, g, b, rm, rv)
        assert max_rel(y, ry) <= 1e-5
        dx, dg, db = h.bn_backward(mode, x, dy, g, sm, si)
        rdx, rdg, rdb = oracle.ref_bn_backward(mode, x, dy, g, b, rsm, rsi)
        assert max_rel(dx, rdx) <= 1e-4 and max_rel(dg, rdg) <= 1e-4 and max_rel(db, rdb) <= 1e-4


def test_batchnorm_invalid_epsilon(lib):
    h = lib.handle()
    x = np.zeros((1, 2, 2, 2), np.float32)
    with pytest.raises(Exception) as e:
        h.bn_forward_train(abi.BN_SPATIAL, x, np.ones(2), np.zeros(2), np.zeros(2), np.ones(2),
                           eps=0.0)
    assert "INVALID_EPSILON" in str(e.value)


@pytest.mark.parametrize("kind", [abi.RELU, abi.LEAKY_RELU, abi.SIGMOID, abi.TANH])
def test_activation(lib, kind):
    rng = np.random.default_rng(kind)
    h = lib.handle()
    x = rng.uniform(-3, 3, (2, 3, 4, 5)).astype(np.float32)
    x[0, 0, 0, :2] = 0.0
    dy = rng.uniform(-1, 1, x.shape).astype(np.float32)
    y = h.activation_forward(kind, 0.3, x)
    want = oracle.activation(kind, 0.3, x)
    assert max_rel(y, want) <= 1e-6
    dx = h.activation_backward(kind, 0.3, x, dy)
    r = oracle.restated()
    g = np.vectorize(lambda v: r.oc_activation_grad(kind, 0.3, float(v)), otypes=[np.float32])(x)
    assert max_rel(dx, g * dy) <= 1e-6
    if kind == abi.RELU:
        assert np.all(dx[0, 0, 0, :2] == 0)  # ReLU'(0) = 0
