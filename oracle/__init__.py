"""Parity oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker
or the timed CPU reference arm — never as a product path. Two oracles live
here:

* ``restated()``: ``oracle/liboracle.so`` built from ``primkit_oracle.c``, a
  plain-C restatement of the reference CPU algorithms (each function cites
  the reference file:line it follows);
* ``reference()``: ``oracle/_ref/libprimkit_ref.so``, the unmodified reference
  implementation compiled from /root/reference sources by
  ``oracle/Makefile.ref`` (plus ``ref_shim.cpp`` exposing its C++-only
  batch-norm / activation entry points). It travels to the GPU box as a
  prebuilt binary; /root/reference itself is never read at run time.

The restatement is pinned against the reference's golden vectors
(tests/golden/) and against ``reference()`` (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libprimkit_ref.so")
REF_SOURCES = "/root/reference/proj"


def build(force: bool = False) -> None:
    """Compile the C restatement and (when the reference sources exist here)
    the reference library. Building the checker is not using it."""
    src = os.path.join(_HERE, "primkit_oracle.c")
    if force or not os.path.exists(RESTATED_SO) or os.path.getmtime(src) > os.path.getmtime(RESTATED_SO):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", RESTATED_SO, src,
                               "-lm"])
    if os.path.isdir(REF_SOURCES):  # make is incremental (shim / source timestamps)
        subprocess.check_call(["make", "-s", "-f", os.path.join(_HERE, "Makefile.ref"),
                               f"-j{os.cpu_count() or 4}"] + (["-B"] if force else []))


class _ConvP(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n", "c", "h", "w", "k", "y", "x", "pad_h", "pad_w",
                                         "str_h", "str_w", "dil_h", "dil_w", "groups")]


_FP = C.POINTER(C.c_float)
_restated = None


def _fp(a):
    return a.ctypes.data_as(_FP)


def restated():
    """The C restatement (ctypes CDLL with typed entry points)."""
    global _restated
    if _restated is None:
        if not os.path.exists(RESTATED_SO):
            build()
        lib = C.CDLL(RESTATED_SO)
        lib.oc_round_bf16.restype = C.c_float
        lib.oc_round_bf16.argtypes = [C.c_float]
        lib.oc_activation.restype = C.c_float
        lib.oc_activation.argtypes = [C.c_int, C.c_float, C.c_float]
        lib.oc_activation_grad.restype = C.c_float
        lib.oc_activation_grad.argtypes = [C.c_int, C.c_float, C.c_float]
        lib.oc_fused_epilogue.restype = C.c_float
        lib.oc_fused_epilogue.argtypes = [C.c_float, C.c_int, C.c_float, C.c_int, C.c_float,
                                          C.c_float, C.c_float, C.c_float, C.c_float, C.c_int,
                                          C.c_float]
        _restated = lib
    return _restated


def _convp(p) -> _ConvP:
    cp = _ConvP()
    for a, b in (("n", "n"), ("c", "c"), ("h", "h"), ("w", "w"), ("k", "k"), ("y", "y"), ("x", "x"),
                 ("pad_h", "pad_h"), ("pad_w", "pad_w"), ("str_h", "stride_h"),
                 ("str_w", "stride_w"), ("dil_h", "dilation_h"), ("dil_w", "dilation_w"),
                 ("groups", "groups")):
        setattr(cp, a, getattr(p, b))
    return cp


def out_hw(p):
    def ext(i, pad, d, f, s):
        span = d * (f - 1) + 1
        return 0 if i + 2 * pad < span else (i + 2 * pad - span) // s + 1
    return (ext(p.h, p.pad_h, p.dilation_h, p.y, p.stride_h),
            ext(p.w, p.pad_w, p.dilation_w, p.x, p.stride_w))


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Vectorised restatement of tensor.cpp:44-54 (RNE, NaN -> quiet NaN)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    nan = np.isnan(a)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    r = np.where(nan, (u.astype(np.uint32) & 0xFFFF0000) | 0x00410000, r).astype(np.uint32)
    return r.view(np.float32)


def conv_forward(p, x, w, bf16=False):
    oh, ow = out_hw(p)
    out = np.zeros((p.n, p.k, oh, ow), np.float32)
    restated().oc_conv_fwd(C.byref(_convp(p)), _fp(np.ascontiguousarray(x, np.float32)),
                           _fp(np.ascontiguousarray(w, np.float32)), _fp(out), int(bf16))
    return out


def conv_backward_data(p, dy, w, bf16=False):
    dx = np.zeros((p.n, p.c, p.h, p.w), np.float32)
    restated().oc_conv_bwd_data(C.byref(_convp(p)), _fp(np.ascontiguousarray(dy, np.float32)),
                                _fp(np.ascontiguousarray(w, np.float32)), _fp(dx), int(bf16))
    return dx


def conv_backward_weights(p, dy, x, bf16=False):
    dw = np.zeros((p.k, p.c // p.groups, p.y, p.x), np.float32)
    restated().oc_conv_bwd_weights(C.byref(_convp(p)), _fp(np.ascontiguousarray(dy, np.float32)),
                                   _fp(np.ascontiguousarray(x, np.float32)), _fp(dw), int(bf16))
    return dw


def winograd_f23(p, x, w, bf16=False):
    oh, ow = out_hw(p)
    out = np.zeros((p.n, p.k, oh, ow), np.float32)
    restated().oc_winograd_f23(C.byref(_convp(p)), _fp(np.ascontiguousarray(x, np.float32)),
                               _fp(np.ascontiguousarray(w, np.float32)), _fp(out), int(bf16))
    return out


def _d4(shape):
    return (C.c_int64 * 4)(*shape)


def bn_forward_train(mode, x, gamma, beta, rmean, rvar, eps=1e-5, momentum=0.1, bf16=False):
    x = np.ascontiguousarray(x, np.float32)
    rm, rv = np.array(rmean, np.float32).ravel(), np.array(rvar, np.float32).ravel()
    ns = rm.size
    y = np.zeros_like(x)
    sm, si = np.zeros(ns, np.float32), np.zeros(ns, np.float32)
    restated().oc_bn_forward_train(mode, _d4(x.shape), _fp(x),
                                   _fp(np.ascontiguousarray(gamma, np.float32).ravel()),
                                   _fp(np.ascontiguousarray(beta, np.float32).ravel()), _fp(rm),
                                   _fp(rv), C.c_float(eps), C.c_float(momentum), _fp(y), _fp(sm),
                                   _fp(si), int(bf16))
    return y, sm, si, rm, rv


def bn_forward_infer(mode, x, gamma, beta, rmean, rvar, eps=1e-5, bf16=False):
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros_like(x)
    f = lambda a: _fp(np.ascontiguousarray(a, np.float32).ravel())  # noqa: E731
    args = [np.ascontiguousarray(a, np.float32).ravel() for a in (gamma, beta, rmean, rvar)]
    restated().oc_bn_forward_infer(mode, _d4(x.shape), _fp(x), *[_fp(a) for a in args],
                                   C.c_float(eps), _fp(y), int(bf16))
    del f
    return y


def bn_backward(mode, x, dy, gamma, smean, sinv, bf16=False):
    x, dy = np.ascontiguousarray(x, np.float32), np.ascontiguousarray(dy, np.float32)
    g = np.ascontiguousarray(gamma, np.float32).ravel()
    dx = np.zeros_like(x)
    dg, db = np.zeros(g.size, np.float32), np.zeros(g.size, np.float32)
    restated().oc_bn_backward(mode, _d4(x.shape), _fp(x), _fp(dy), _fp(g),
                              _fp(np.ascontiguousarray(smean, np.float32)),
                              _fp(np.ascontiguousarray(sinv, np.float32)), _fp(dx), _fp(dg),
                              _fp(db), int(bf16))
    return dx, dg, db


def activation(kind, alpha, x):
    f = np.vectorize(lambda v: restated().oc_activation(kind, alpha, float(v)), otypes=[np.float32])
    return f(np.asarray(x, np.float32))


def conv_ref_f64(p, x, w):
    """Independent f64 scatter-form reference (structure of the reference's
    tests/test_util.hpp:37-116 conv_ref), vectorised over (n, k) with numpy."""
    oh, ow = out_hw(p)
    out = np.zeros((p.n, p.k, oh, ow), np.float64)
    cg, kg = p.c // p.groups, p.k // p.groups
    x = x.astype(np.float64)
    w = w.astype(np.float64)
    for g in range(p.groups):
        for yy in range(p.y):
            for xx in range(p.x):
                for o_h in range(oh):
                    ih = o_h * p.stride_h - p.pad_h + yy * p.dilation_h
                    if ih < 0 or ih >= p.h:
                        continue
                    iws = np.arange(ow) * p.stride_w - p.pad_w + xx * p.dilation_w
                    ok = (iws >= 0) & (iws < p.w)
                    if not ok.any():
                        continue
                    xs = x[:, g * cg:(g + 1) * cg, ih, :][:, :, iws[ok]]          # n, cg, q
                    ws = w[g * kg:(g + 1) * kg, :, yy, xx]                         # kg, cg
                    out[:, g * kg:(g + 1) * kg, o_h, ok] += np.einsum("ncq,kc->nkq", xs, ws)
    return out


# ---- sampled direct formulas on the device layout (full-size parity) -------

class _DevG(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n", "c", "h", "w", "k", "r", "s", "p", "q", "pad_h",
                                         "pad_w", "str_h", "str_w", "dil_h", "dil_w", "xp", "yp",
                                         "fp", "bf16")]


def dev_geom(p, bf16=True) -> _DevG:
    """Device-layout geometry of a (groups = 1, convolution-mode) problem:
    activations NHWC with channel pitch roundup(C, 8), filter [K][R][S][pitch(C)]."""
    oh, ow = out_hw(p)
    pit = lambda c: (c + 7) // 8 * 8  # noqa: E731
    return _DevG(p.n, p.c, p.h, p.w, p.k, p.y, p.x, oh, ow, p.pad_h, p.pad_w, p.stride_h,
                 p.stride_w, p.dilation_h, p.dilation_w, pit(p.c), pit(p.k), pit(p.c), int(bf16))


def _vp(a):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def sample_forward(p, x, w, idx, bf16=True):
    """f64 forward outputs at idx (ns x 4: n, k, oh, ow); x, w in the device
    layout (uint16 bf16 bits or float32). Restates conv.cpp:99-133."""
    idx = np.ascontiguousarray(idx, np.int64)
    out = np.zeros(len(idx), np.float64)
    lib = restated()
    lib.oc_sample_fwd(C.byref(dev_geom(p, bf16)), _vp(x), _vp(w), _vp(idx), C.c_int64(len(idx)), _vp(out))
    return out


def sample_backward_data(p, dy, w, idx, bf16=True):
    """f64 dX at idx (ns x 4: n, c, h, w). Restates conv.cpp:702-799."""
    idx = np.ascontiguousarray(idx, np.int64)
    out = np.zeros(len(idx), np.float64)
    restated().oc_sample_dgrad(C.byref(dev_geom(p, bf16)), _vp(dy), _vp(w), _vp(idx),
                               C.c_int64(len(idx)), _vp(out))
    return out


def sample_backward_weights(p, dy, x, ks, taps, bf16=True):
    """f64 dW on the grid ks x taps (taps: nt x 3 = r, s, c) -> [len(ks), nt].
    Restates conv.cpp:801-873."""
    ks = np.ascontiguousarray(ks, np.int64)
    taps = np.ascontiguousarray(taps, np.int64)
    out = np.zeros((len(ks), len(taps)), np.float64)
    restated().oc_sample_wgrad(C.byref(dev_geom(p, bf16)), _vp(dy), _vp(x), _vp(ks),
                               C.c_int64(len(ks)), _vp(taps), C.c_int64(len(taps)), _vp(out))
    return out


def bn_stats_device(x, c, eps=1e-5, bf16=True):
    """Spatial BN batch statistics (primitives.cpp:61-96) of a device-layout
    tensor x (... x pitch): (mean f32, invstd f32, biased var f64) per channel."""
    pitch = x.shape[-1]
    rows = x.size // pitch
    mean, inv = np.zeros(c, np.float32), np.zeros(c, np.float32)
    var = np.zeros(c, np.float64)
    restated().oc_bn_stats_dev(_vp(np.ascontiguousarray(x)), C.c_int64(rows), C.c_int64(c),
                               C.c_int64(pitch), C.c_int64(int(bf16)), C.c_float(eps), _vp(mean),
                               _vp(inv), _vp(var))
    return mean, inv, var


# ---- pooling / softmax (primitives.cpp:204-370) --------------------------------

_I64 = C.POINTER(C.c_int64)


def _i64(a):
    return (C.c_int64 * len(a))(*[int(v) for v in a])


def pool_out_hw(dims, win, pad, stride):
    return ((dims[2] + 2 * pad[0] - win[0]) // stride[0] + 1, (dims[3] + 2 * pad[1] - win[1]) // stride[1] + 1)


def pool_forward(kind, x, win, pad, stride, bf16=False):
    """(y, indices) of the restated reference pooling (kind 0 max, 1 avg)."""
    x = np.ascontiguousarray(x, np.float32)
    oh, ow = pool_out_hw(x.shape, win, pad, stride)
    y = np.zeros((x.shape[0], x.shape[1], oh, ow), np.float32)
    idx = np.zeros(y.shape, np.int64)
    restated().oc_pool_fwd(kind, _i64(x.shape), _i64(win), _i64(pad), _i64(stride), _fp(x), _fp(y),
                           idx.ctypes.data_as(_I64), int(bf16))
    return y, idx


def pool_backward(kind, in_dims, dy, idx, win, pad, stride, bf16=False):
    dy = np.ascontiguousarray(dy, np.float32)
    idx = np.ascontiguousarray(idx, np.int64)
    dx = np.zeros(in_dims, np.float32)
    restated().oc_pool_bwd(kind, _i64(in_dims), _i64(win), _i64(pad), _i64(stride), _fp(dy),
                           idx.ctypes.data_as(_I64), _fp(dx), int(bf16))
    return dx


def _split(shape, axis):
    outer = int(np.prod(shape[:axis])) if axis else 1
    inner = int(np.prod(shape[axis + 1:])) if axis + 1 < len(shape) else 1
    return outer, shape[axis], inner


def softmax_forward(x, axis, bf16=False):
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros_like(x)
    o, a, i = _split(x.shape, axis)
    restated().oc_softmax_fwd(C.c_int64(o), C.c_int64(a), C.c_int64(i), _fp(x), _fp(y), int(bf16))
    return y


def softmax_backward(y, dy, axis, bf16=False):
    y, dy = np.ascontiguousarray(y, np.float32), np.ascontiguousarray(dy, np.float32)
    dx = np.zeros_like(y)
    o, a, i = _split(y.shape, axis)
    restated().oc_softmax_bwd(C.c_int64(o), C.c_int64(a), C.c_int64(i), _fp(y), _fp(dy), _fp(dx), int(bf16))
    return dx


def ref_pool_forward(kind, x, win, pad, stride, bf16=False):
    L = reference().lib
    x = np.ascontiguousarray(x, np.float32)
    oh, ow = pool_out_hw(x.shape, win, pad, stride)
    y = np.zeros((x.shape[0], x.shape[1], oh, ow), np.float32)
    idx = np.zeros(y.shape, np.int64)
    ref_check(L.ref_pooling_forward(kind, _i64(win), _i64(pad), _i64(stride), _i64(x.shape), int(bf16), _fp(x),
                                    _fp(y), idx.ctypes.data_as(_I64)))
    return y, idx


def ref_pool_backward(kind, in_dims, dy, idx, win, pad, stride, bf16=False):
    L = reference().lib
    dx = np.zeros(in_dims, np.float32)
    ref_check(L.ref_pooling_backward(kind, _i64(win), _i64(pad), _i64(stride), _i64(in_dims), int(bf16),
                                     _fp(np.ascontiguousarray(dy, np.float32)),
                                     np.ascontiguousarray(idx, np.int64).ctypes.data_as(_I64), _fp(dx)))
    return dx


def ref_softmax_forward(x, axis, bf16=False):
    L = reference().lib
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros_like(x)
    ref_check(L.ref_softmax_forward(x.ndim, _i64(x.shape), int(bf16), C.c_int64(axis), _fp(x), _fp(y)))
    return y


def ref_softmax_backward(y, dy, axis, bf16=False):
    L = reference().lib
    y, dy = np.ascontiguousarray(y, np.float32), np.ascontiguousarray(dy, np.float32)
    dx = np.zeros_like(y)
    ref_check(L.ref_softmax_backward(y.ndim, _i64(y.shape), int(bf16), C.c_int64(axis), _fp(y), _fp(dy), _fp(dx)))
    return dx


# ---- the unmodified reference library -------------------------------------

def reference_available() -> bool:
    return os.path.exists(REF_SO)


_ref = None


def reference():
    """(Library, shim) for oracle/_ref/libprimkit_ref.so, or None if absent."""
    global _ref
    if _ref is None:
        if not reference_available():
            return None
        from paper_1910_00078_b200.primkit import Library
        lib = Library(REF_SO, extended=False)
        s = lib.lib
        I64P = C.POINTER(C.c_int64)
        s.ref_bn_forward_train.argtypes = [C.c_int, I64P, C.c_int] + [_FP] * 5 + [
            C.c_float, C.c_float] + [_FP] * 3
        s.ref_bn_forward_infer.argtypes = [C.c_int, I64P, C.c_int] + [_FP] * 5 + [C.c_float, _FP]
        s.ref_bn_backward.argtypes = [C.c_int, I64P, C.c_int] + [_FP] * 6 + [C.c_float] + [_FP] * 3
        s.ref_activation_forward.argtypes = [C.c_int, C.c_float, I64P, C.c_int, _FP, _FP]
        s.ref_activation_backward.argtypes = [C.c_int, C.c_float, I64P, C.c_int, _FP, _FP, _FP]
        s.ref_round_bf16.restype = C.c_float
        s.ref_round_bf16.argtypes = [C.c_float]
        s.ref_shim_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


def ref_check(st):
    if st != 0:
        raise RuntimeError(f"reference shim status {st}: "
                           f"{reference().lib.ref_shim_last_error().decode()}")


def ref_bn_forward_train(mode, x, gamma, beta, rmean, rvar, eps=1e-5, momentum=0.1, bf16=False):
    L = reference().lib
    x = np.ascontiguousarray(x, np.float32)
    rm, rv = np.array(rmean, np.float32).ravel(), np.array(rvar, np.float32).ravel()
    y = np.zeros_like(x)
    sm, si = np.zeros(rm.size, np.float32), np.zeros(rm.size, np.float32)
    ref_check(L.ref_bn_forward_train(mode, _d4(x.shape), int(bf16), _fp(x),
                                     _fp(np.ascontiguousarray(gamma, np.float32).ravel()),
                                     _fp(np.ascontiguousarray(beta, np.float32).ravel()), _fp(rm),
                                     _fp(rv), C.c_float(eps), C.c_float(momentum), _fp(y), _fp(sm),
                                     _fp(si)))
    return y, sm, si, rm, rv


def ref_bn_backward(mode, x, dy, gamma, beta, smean, sinv, eps=1e-5, bf16=False):
    L = reference().lib
    x, dy = np.ascontiguousarray(x, np.float32), np.ascontiguousarray(dy, np.float32)
    g = np.ascontiguousarray(gamma, np.float32).ravel()
    dx = np.zeros_like(x)
    dg, db = np.zeros(g.size, np.float32), np.zeros(g.size, np.float32)
    ref_check(L.ref_bn_backward(mode, _d4(x.shape), int(bf16), _fp(x), _fp(dy), _fp(g),
                                _fp(np.ascontiguousarray(beta, np.float32).ravel()),
                                _fp(np.ascontiguousarray(smean, np.float32)),
                                _fp(np.ascontiguousarray(sinv, np.float32)), C.c_float(eps),
                                _fp(dx), _fp(dg), _fp(db)))
    return dx, dg, db
