"""Python host binding of the primkit C ABI.

Thin ctypes layer over ``lib/libprimkit.so`` (the B200 library). The same
wrapper class also drives any library exporting the reference ABI (the
parity tests point it at the reference build in ``oracle/_ref``), so a test
reads exactly like the reference's own C ABI tests
(/root/reference/proj/tests/test_capi.cpp).

There is no Python or CPU compute path here: every numeric call goes
through the shared library, and loading fails loudly if it was not built.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import abi

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libprimkit.so")


class PrimkitError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        self.name = abi.STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {message}")


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _fp(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(abi.FP)


def _dims(d) -> C.Array:
    return (C.c_int64 * 4)(*[int(v) for v in d])


def problem(n=1, c=1, h=1, w=1, k=1, y=1, x=1, pad=0, stride=1, dilation=1, groups=1,
            direction=abi.FORWARD, mode=abi.CONVOLUTION, etype=abi.F32, pad_h=None, pad_w=None,
            stride_h=None, stride_w=None, dilation_h=None, dilation_w=None) -> abi.ConvProblem:
    p = abi.ConvProblem()
    p.n, p.c, p.h, p.w, p.k, p.y, p.x = n, c, h, w, k, y, x
    p.pad_h = pad if pad_h is None else pad_h
    p.pad_w = pad if pad_w is None else pad_w
    p.stride_h = stride if stride_h is None else stride_h
    p.stride_w = stride if stride_w is None else stride_w
    p.dilation_h = dilation if dilation_h is None else dilation_h
    p.dilation_w = dilation if dilation_w is None else dilation_w
    p.groups, p.direction, p.mode, p.etype = groups, direction, mode, etype
    return p


@dataclass
class AlgoPerf:
    solver_name: str
    algo: int
    time_ms: float
    workspace_bytes: int


class Library:
    """A loaded primkit ABI library (ours or the reference oracle)."""

    def __init__(self, path: str, extended: bool = True):
        if not os.path.exists(path):
            raise ImportError(f"primkit library not built: {path} "
                              "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        self.path = path
        self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        abi.bind(self.lib, (abi.SECTION1, abi.SECTION2) if extended else (abi.SECTION1,))
        self.extended = extended

    # -- error plumbing --
    def last_error(self) -> str:
        return (self.lib.primkit_last_error() or b"").decode()

    def check(self, status: int) -> None:
        if status != 0:
            raise PrimkitError(status, self.last_error())

    def status(self, fn, *args) -> int:
        """Raw status of a call (for tests asserting error codes)."""
        return getattr(self.lib, fn)(*args)

    # -- problem queries --
    def problem_key(self, p: abi.ConvProblem) -> str:
        buf = C.create_string_buffer(256)
        self.check(self.lib.primkit_problem_key(C.byref(p), buf, 256))
        return buf.value.decode()

    def output_dims(self, p: abi.ConvProblem) -> list[int]:
        d = (C.c_int64 * 4)()
        self.check(self.lib.primkit_conv_output_dims(C.byref(p), d))
        return list(d)

    def handle(self) -> "Handle":
        return Handle(self)

    def fusion_plan(self, dims, etype=abi.F32) -> "FusionPlan":
        return FusionPlan(self, dims, etype)

    def channel_pitch(self, c: int) -> int:
        return int(self.lib.primkit_channel_pitch(c))


def operand_shapes(lib: Library, p: abi.ConvProblem):
    """(a, b, result) NCHW shapes for a problem's direction (primkit_c.cpp:73-105)."""
    inp = (p.n, p.c, p.h, p.w)
    flt = (p.k, p.c // p.groups, p.y, p.x) if p.mode == abi.CONVOLUTION else (
        p.c, p.k // p.groups, p.y, p.x)
    fwd = abi.ConvProblem.from_buffer_copy(p)
    fwd.direction = abi.FORWARD
    out = tuple(lib.output_dims(fwd))
    if p.direction == abi.FORWARD:
        return inp, flt, out
    if p.direction == abi.BACKWARD_DATA:
        return out, flt, inp
    return out, inp, flt


class Handle:
    def __init__(self, lib: Library):
        self.L = lib
        self.ptr = C.c_void_p()
        lib.check(lib.lib.primkit_handle_create(C.byref(self.ptr)))

    def close(self):
        if self.ptr:
            self.L.lib.primkit_handle_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _c(self, name, *args):
        self.L.check(getattr(self.L.lib, name)(self.ptr, *args))

    def use_fake_clock(self):
        self._c("primkit_handle_use_fake_clock")

    def now_ms(self) -> float:
        v = C.c_double()
        self._c("primkit_handle_now_ms", C.byref(v))
        return v.value

    def set_cache_dir(self, d: str):
        self._c("primkit_handle_set_cache_dir", d.encode())

    def counters(self) -> tuple[int, int, int]:
        c = abi.Counters()
        self._c("primkit_handle_counters", C.byref(c))
        return c.gemm_calls, c.scalar_muls, c.buffer_roundtrips

    def reset_counters(self):
        self._c("primkit_handle_reset_counters")

    def set_seed(self, s: int):
        self._c("primkit_handle_set_seed", C.c_uint64(s))

    def solver_names(self) -> list[str]:
        n = C.c_int()
        self._c("primkit_solver_count", C.byref(n))
        out = []
        for i in range(n.value):
            buf = C.create_string_buffer(64)
            self._c("primkit_solver_name", i, buf, 64)
            out.append(buf.value.decode())
        return out

    def is_applicable(self, solver: str, p) -> bool:
        v = C.c_int()
        self._c("primkit_solver_is_applicable", solver.encode(), C.byref(p), C.byref(v))
        return bool(v.value)

    def is_tunable(self, solver: str) -> bool:
        v = C.c_int()
        self._c("primkit_solver_is_tunable", solver.encode(), C.byref(v))
        return bool(v.value)

    def workspace_bytes(self, solver: str, p) -> int:
        v = C.c_uint64()
        self._c("primkit_solver_workspace_bytes", solver.encode(), C.byref(p), C.byref(v))
        return v.value

    def find(self, p, a, b, workspace_bytes: int, capacity: int = 8):
        a, b = _f32(a), _f32(b)
        res = (abi.AlgoPerf * max(capacity, 1))()
        cnt = C.c_int()
        self._c("primkit_find_convolution", C.byref(p), _fp(a), _fp(b), workspace_bytes, res,
                capacity, C.byref(cnt))
        rows = [AlgoPerf(r.solver_name.decode(), r.algo, r.time_ms, r.workspace_bytes)
                for r in res[:min(capacity, cnt.value)]]
        return rows, cnt.value

    def conv_run(self, p, solver: str | None, a, b, workspace_bytes: int | None = None):
        a, b = _f32(a), _f32(b)
        if workspace_bytes is None:
            # exactly what the solver asks for (the reference allocates the
            # caller's workspace size, so never pass a huge default)
            names = [solver] if solver else [s for s in self.solver_names()
                                             if self.is_applicable(s, p)][:1]
            workspace_bytes = max([self.workspace_bytes(s, p) for s in names] + [0])
        out = np.zeros(operand_shapes(self.L, p)[2], dtype=np.float32)
        self._c("primkit_conv_run", C.byref(p), None if solver is None else solver.encode(),
                _fp(a), _fp(b), _fp(out), C.c_size_t(workspace_bytes))
        return out

    def tune(self, p, solver: str, budget: int = 0, exhaustive: bool = False) -> int:
        ev = C.c_int64()
        self._c("primkit_tune", C.byref(p), solver.encode(), budget, int(exhaustive), C.byref(ev))
        return ev.value

    def perfdb_save(self, path: str):
        self._c("primkit_perfdb_save", path.encode())

    def perfdb_load(self, path: str):
        self._c("primkit_perfdb_load", path.encode())

    # -- batch-norm / activation (B200 ABI section 2) --
    def bn_forward_train(self, mode, x, gamma, beta, rmean, rvar, eps=1e-5, momentum=0.1,
                         etype=abi.F32):
        x = _f32(x)
        g, b = _f32(gamma).ravel(), _f32(beta).ravel()
        rm, rv = _f32(rmean).ravel().copy(), _f32(rvar).ravel().copy()
        ns = g.size
        y = np.zeros_like(x)
        sm, si = np.zeros(ns, np.float32), np.zeros(ns, np.float32)
        self._c("primkit_batchnorm_forward_train", mode, _dims(x.shape), etype, _fp(x), _fp(g),
                _fp(b), _fp(rm), _fp(rv), C.c_float(eps), C.c_float(momentum), _fp(y), _fp(sm),
                _fp(si))
        return y, sm, si, rm, rv

    def bn_forward_infer(self, mode, x, gamma, beta, rmean, rvar, eps=1e-5, etype=abi.F32):
        x = _f32(x)
        y = np.zeros_like(x)
        self._c("primkit_batchnorm_forward_infer", mode, _dims(x.shape), etype, _fp(x),
                _fp(_f32(gamma).ravel()), _fp(_f32(beta).ravel()), _fp(_f32(rmean).ravel()),
                _fp(_f32(rvar).ravel()), C.c_float(eps), _fp(y))
        return y

    def bn_backward(self, mode, x, dy, gamma, saved_mean, saved_invstd, etype=abi.F32):
        x, dy = _f32(x), _f32(dy)
        g = _f32(gamma).ravel()
        dx = np.zeros_like(x)
        dg, db = np.zeros(g.size, np.float32), np.zeros(g.size, np.float32)
        self._c("primkit_batchnorm_backward", mode, _dims(x.shape), etype, _fp(x), _fp(dy),
                _fp(g), _fp(_f32(saved_mean)), _fp(_f32(saved_invstd)), _fp(dx), _fp(dg), _fp(db))
        return dx, dg, db

    def activation_forward(self, kind, alpha, x, etype=abi.F32):
        x = _f32(x)
        y = np.zeros_like(x)
        self._c("primkit_activation_forward", kind, C.c_float(alpha), _dims(x.shape), etype,
                _fp(x), _fp(y))
        return y

    def activation_backward(self, kind, alpha, x, dy, etype=abi.F32):
        x, dy = _f32(x), _f32(dy)
        dx = np.zeros_like(x)
        self._c("primkit_activation_backward", kind, C.c_float(alpha), _dims(x.shape), etype,
                _fp(x), _fp(dy), _fp(dx))
        return dx

    def kernel_launches(self) -> int:
        v = C.c_uint64()
        self._c("primkit_handle_kernel_launches", C.byref(v))
        return v.value

    def last_device_ms(self) -> float:
        v = C.c_double()
        self._c("primkit_handle_last_device_ms", C.byref(v))
        return v.value

    def last_kernel(self) -> str:
        buf = C.create_string_buffer(128)
        self._c("primkit_handle_last_kernel", buf, 128)
        return buf.value.decode()

    def pooling_forward(self, kind, x, window, pad=(0, 0), stride=None, etype=abi.F32):
        """(y, indices) — reference pooling_forward (primitives.cpp:204-260)."""
        x = _f32(x)
        stride = window if stride is None else stride
        od = (C.c_int64 * 4)()
        i64 = lambda v: (C.c_int64 * len(v))(*v)  # noqa: E731
        self.L.check(self.L.lib.primkit_pooling_output_dims(i64(window), i64(pad), i64(stride),
                                                            _dims(x.shape), od))
        y = np.zeros(list(od), np.float32)
        idx = np.zeros(list(od), np.int64)
        self._c("primkit_pooling_forward", kind, i64(window), i64(pad), i64(stride), _dims(x.shape), etype,
                _fp(x), _fp(y), idx.ctypes.data_as(C.POINTER(C.c_int64)))
        return y, idx

    def pooling_backward(self, kind, in_dims, dy, indices, window, pad=(0, 0), stride=None, etype=abi.F32):
        dy = _f32(dy)
        stride = window if stride is None else stride
        i64 = lambda v: (C.c_int64 * len(v))(*v)  # noqa: E731
        dx = np.zeros(in_dims, np.float32)
        idx = None if indices is None else np.ascontiguousarray(indices, np.int64)
        self._c("primkit_pooling_backward", kind, i64(window), i64(pad), i64(stride), _dims(in_dims), etype,
                _fp(dy), None if idx is None else idx.ctypes.data_as(C.POINTER(C.c_int64)), _fp(dx))
        return dx

    def softmax_forward(self, x, axis, etype=abi.F32):
        x = _f32(x)
        y = np.zeros_like(x)
        self._c("primkit_softmax_forward", x.ndim, (C.c_int64 * x.ndim)(*x.shape), etype, axis, _fp(x), _fp(y))
        return y

    def softmax_backward(self, y, dy, axis, etype=abi.F32):
        y, dy = _f32(y), _f32(dy)
        dx = np.zeros_like(y)
        self._c("primkit_softmax_backward", y.ndim, (C.c_int64 * y.ndim)(*y.shape), etype, axis, _fp(y),
                _fp(dy), _fp(dx))
        return dx

    def plan_cache_stats(self) -> tuple[int, int, int]:
        """(builds, memory_hits, disk_hits) of the handle's plan cache."""
        v = [C.c_uint64() for _ in range(3)]
        self._c("primkit_handle_plan_cache_stats", *[C.byref(x) for x in v])
        return tuple(x.value for x in v)

    def device_workspace(self, p, solver: str | None) -> int:
        """Device scratch of the plan for (p, solver); one cached_build."""
        v = C.c_uint64()
        self._c("primkit_conv_device_workspace", C.byref(p), None if solver is None else solver.encode(),
                C.byref(v))
        return v.value

    def last_variant(self) -> str:
        buf = C.create_string_buffer(1024)
        self._c("primkit_handle_last_variant", buf, 1024)
        return buf.value.decode()

    def tune_kernels(self, p, solver: str, budget: int = 0) -> tuple[str, float, float]:
        """B200 kernel-choice search (primkit_tune_kernels): (best values,
        heuristic median ms, best median ms); the best is stored in the perf-db."""
        buf = C.create_string_buffer(64)
        d, b = C.c_double(), C.c_double()
        self._c("primkit_tune_kernels", C.byref(p), solver.encode(), budget, buf, 64, C.byref(d),
                C.byref(b))
        return buf.value.decode(), d.value, b.value

    def kernel_config(self, p, solver: str) -> str:
        buf = C.create_string_buffer(64)
        self._c("primkit_plan_kernel_config", C.byref(p), solver.encode(), buf, 64)
        return buf.value.decode()

    def load_system_db(self, path: str | None):
        self._c("primkit_handle_load_system_db", (path or "").encode())

    def system_db(self) -> tuple[str, int]:
        buf = C.create_string_buffer(4096)
        n = C.c_uint64()
        self._c("primkit_handle_system_db", buf, 4096, C.byref(n))
        return buf.value.decode(), n.value


class FusionPlan:
    def __init__(self, lib: Library, dims, etype=abi.F32):
        self.L = lib
        self.ptr = C.c_void_p()
        self.dims = tuple(int(v) for v in dims)
        lib.check(lib.lib.primkit_fusion_plan_create(_dims(dims), etype, C.byref(self.ptr)))

    def close(self):
        if self.ptr:
            self.L.lib.primkit_fusion_plan_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def st(self, name, *args) -> int:
        return getattr(self.L.lib, name)(self.ptr, *args)

    def add_conv(self, filter_dims, pad=0, stride=1, groups=1, algo="Direct", pad_w=None,
                 stride_w=None):
        return self.st("primkit_fusion_add_conv", _dims(filter_dims), pad,
                       pad if pad_w is None else pad_w, stride,
                       stride if stride_w is None else stride_w, groups, abi.ALGO[algo])

    def add_bias(self, channels):
        return self.st("primkit_fusion_add_bias", channels)

    def add_batchnorm(self, mode=abi.BN_SPATIAL):
        return self.st("primkit_fusion_add_batchnorm", mode)

    def add_activation(self, kind, alpha=0.0):
        return self.st("primkit_fusion_add_activation", kind, C.c_float(alpha))

    def compile(self, handle: Handle) -> int:
        return self.L.lib.primkit_fusion_compile(handle.ptr, self.ptr)

    def output_dims(self):
        d = (C.c_int64 * 4)()
        self.L.check(self.st("primkit_fusion_output_dims", d))
        return list(d)

    def set_args(self, filter=None, bias=None, gamma=None, beta=None, mean=None, var=None,
                 eps=1e-5, act_alpha=None):
        keep = [None if v is None else _f32(v) for v in (filter, bias, gamma, beta, mean, var)]
        alpha = None if act_alpha is None else C.byref(C.c_float(act_alpha))
        self.L.check(self.st("primkit_fusion_set_args", *[_fp(v) for v in keep], C.c_float(eps),
                             alpha))

    def execute(self, handle: Handle, x, unfused=False, check=True):
        x = _f32(x)
        out = np.zeros(self.output_dims(), np.float32)
        st = self.L.lib.primkit_fusion_execute(handle.ptr, self.ptr, _fp(x), _fp(out),
                                               int(unfused))
        if check:
            self.L.check(st)
            return out
        return st, out


_product: Library | None = None


def library() -> Library:
    """The B200 library (loaded once; raises ImportError if not built)."""
    global _product
    if _product is None:
        _product = Library(LIB_PATH)
    return _product
