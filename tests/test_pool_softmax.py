"""Pooling and softmax (reference primitives.cpp:204-370)
through the C ABI. GPU results are compared with the oracle restatement,
which tests/test_oracle.py pins bit-for-bit against the reference library:
pooling values, argmax indices and gradients bit-exact (f32 and bf16);
softmax within 1e-6 (f32; the row reduction order differs) / one bf16 ulp.
Argument validation happens on the host, so its tests run without a GPU."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi

POOL_CASES = [
    ((2, 64, 112, 112), (3, 3), (1, 1), (2, 2)),   # ResNet-50 stem max-pool
    ((4, 2048, 7, 7), (7, 7), (0, 0), (1, 1)),     # ResNet-50 global average pool
    ((2, 3, 9, 8), (3, 2), (1, 0), (1, 2)),        # overlapping, C not a multiple of 8
    ((1, 5, 3, 3), (5, 5), (2, 2), (3, 3)),        # windows larger than the image
    ((3, 16, 6, 5), (2, 2), (0, 0), (2, 2)),
]


def _i64(v):
    return (C.c_int64 * len(v))(*v)


def test_pooling_rejects_bad_descriptor(lib):
    with lib.handle() as h:
        x = np.zeros((1, 1, 4, 4), np.float32)
        y = np.zeros((1, 1, 2, 2), np.float32)
        st = lib.lib.primkit_pooling_forward(h.ptr, abi.POOL_MAX, _i64((0, 2)), _i64((0, 0)), _i64((2, 2)),
                                             _i64(x.shape), abi.F32, x.ctypes.data_as(abi.FP),
                                             y.ctypes.data_as(abi.FP), None)
        assert st == abi.STATUS_CODE["INVALID_VALUE"] and "bad pooling descriptor" in lib.last_error()
        st = lib.lib.primkit_pooling_forward(h.ptr, abi.POOL_MAX, _i64((5, 5)), _i64((0, 0)), _i64((1, 1)),
                                             _i64(x.shape), abi.F32, x.ctypes.data_as(abi.FP),
                                             y.ctypes.data_as(abi.FP), None)
        assert st == abi.STATUS_CODE["INVALID_SHAPE"] and "below 1" in lib.last_error()


def test_pooling_output_dims(lib):
    od = (C.c_int64 * 4)()
    lib.check(lib.lib.primkit_pooling_output_dims(_i64((3, 3)), _i64((1, 1)), _i64((2, 2)),
                                                  _i64((32, 64, 112, 112)), od))
    assert list(od) == [32, 64, 56, 56]


def test_softmax_rejects_bad_axis(lib):
    with lib.handle() as h:
        x = np.zeros((2, 3), np.float32)
        st = lib.lib.primkit_softmax_forward(h.ptr, 2, _i64(x.shape), abi.F32, 2, x.ctypes.data_as(abi.FP),
                                             x.ctypes.data_as(abi.FP))
        assert st == abi.STATUS_CODE["INVALID_AXIS"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", POOL_CASES, ids=lambda c: "x".join(map(str, c[0])))
@pytest.mark.parametrize("kind", [abi.POOL_MAX, abi.POOL_AVG], ids=["max", "avg"])
@pytest.mark.parametrize("etype", [abi.F32, abi.BF16], ids=["f32", "bf16"])
def test_pooling_matches_reference(lib, case, kind, etype):
    dims, win, pad, stride = case
    bf = etype == abi.BF16
    rng = np.random.default_rng(31)
    x = rng.uniform(-1, 1, dims).astype(np.float32)
    x[:, :, 0, :2] = 0.25  # ties
    if bf:
        x = oracle.round_bf16(x)
    with lib.handle() as h:
        y, idx = h.pooling_forward(kind, x, win, pad, stride, etype)
        yo, idxo = oracle.pool_forward(kind, x, win, pad, stride, bf)
        assert np.array_equal(y, yo)
        assert np.array_equal(idx, idxo)
        dy = rng.uniform(-1, 1, y.shape).astype(np.float32)
        if bf:
            dy = oracle.round_bf16(dy)
        dx = h.pooling_backward(kind, dims, dy, idx if kind == abi.POOL_MAX else None, win, pad, stride, etype)
        dxo = oracle.pool_backward(kind, dims, dy, idxo, win, pad, stride, bf)
        assert np.array_equal(dx, dxo)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,axis", [((256, 1000), 1), ((8, 21, 7, 7), 1), ((5, 33), 0), ((3, 4, 130), 2)])
@pytest.mark.parametrize("etype", [abi.F32, abi.BF16], ids=["f32", "bf16"])
def test_softmax_matches_reference(lib, shape, axis, etype):
    bf = etype == abi.BF16
    rng = np.random.default_rng(32)
    x = rng.uniform(-6, 6, shape).astype(np.float32)
    if bf:
        x = oracle.round_bf16(x)
    tol = 2.0 ** -7 if bf else 1e-6
    with lib.handle() as h:
        y = h.softmax_forward(x, axis, etype)
        yo = oracle.softmax_forward(x, axis, bf)
        assert np.max(np.abs(y - yo) / np.maximum(np.abs(yo), 1e-30)) <= tol
        np.testing.assert_allclose(y.sum(axis=axis), 1.0, rtol=0, atol=1e-2 if bf else 1e-5)
        dy = rng.uniform(-1, 1, shape).astype(np.float32)
        if bf:
            dy = oracle.round_bf16(dy)
        dx = h.softmax_backward(yo, dy, axis, etype)
        dxo = oracle.softmax_backward(yo, dy, axis, bf)
        assert np.max(np.abs(dx - dxo)) <= tol * max(1.0, float(np.max(np.abs(dxo))))
