"""Host logic bit-exact against the reference: problem keys, shape algebra and
error statuses, the solver registry (applicability, tunability, workspace
requests), perf-db files, and the fusion metadata-graph verdicts.

Known answers are the reference's own test vectors (file:line cited); the
sweeps compare this library with the unmodified reference library
(oracle/_ref) call by call. None of this touches a GPU."""
import itertools
import os

import numpy as np
import pytest

from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import PrimkitError, problem

SOLVERS = ["Im2colGemm", "Direct", "Winograd", "FFT", "ImplicitGemm"]


def test_problem_key_known_answers(lib):
    # test_solver.cpp:44-65 / test_capi.cpp:66-81
    p = problem(n=32, c=3, h=224, w=224, k=64, y=7, x=7, pad=3, stride=2)
    assert lib.problem_key(p) == "32-3-224-224-64-7-7-3-3-2-2-1-1-1-F-C-f32"
    p.direction, p.etype = abi.BACKWARD_WEIGHTS, abi.BF16
    assert lib.problem_key(p).endswith("-BW-C-bf16")
    p.direction, p.mode = abi.BACKWARD_DATA, abi.TRANSPOSE
    assert lib.problem_key(p).endswith("-BD-T-bf16")


def test_problem_key_buffer_too_small(lib):
    import ctypes as C
    p = problem(n=32, c=3, h=224, w=224, k=64, y=7, x=7, pad=3, stride=2)
    buf = C.create_string_buffer(4)
    assert lib.lib.primkit_problem_key(C.byref(p), buf, 4) == abi.STATUS_CODE["INVALID_VALUE"]
    assert lib.last_error()


def test_output_dims_known_answers(lib):
    # test_conv.cpp:49-62, test_capi.cpp:83-100
    assert lib.output_dims(problem(n=1, c=1, h=5, w=5, k=1, y=3, x=3)) == [1, 1, 3, 3]
    assert lib.output_dims(problem(n=32, c=3, h=224, w=224, k=64, y=7, x=7, pad=3, stride=2)) == [
        32, 64, 112, 112]
    assert lib.output_dims(problem(n=1, c=1, h=9, w=9, k=1, y=3, x=3, dilation=2)) == [1, 1, 5, 5]
    assert lib.output_dims(problem(n=1, c=4, h=7, w=7, k=2, y=3, x=3, pad=1, stride=2,
                                   mode=abi.TRANSPOSE)) == [1, 2, 13, 13]
    p = problem(n=1, c=4, h=8, w=8, k=4, y=3, x=3, pad=1, stride=2)
    assert lib.output_dims(p) == [1, 4, 4, 4]
    p.groups = 3
    with pytest.raises(PrimkitError) as e:
        lib.output_dims(p)
    assert e.value.name == "GROUP_MISMATCH"


def _random_problems(n, seed):
    r = np.random.default_rng(seed)
    for _ in range(n):
        yield problem(
            n=int(r.integers(1, 4)), c=int(r.integers(1, 9)), h=int(r.integers(1, 12)),
            w=int(r.integers(1, 12)), k=int(r.integers(1, 9)), y=int(r.integers(1, 6)),
            x=int(r.integers(1, 6)), pad_h=int(r.integers(0, 3)), pad_w=int(r.integers(0, 3)),
            stride_h=int(r.integers(0, 4)), stride_w=int(r.integers(1, 4)),
            dilation_h=int(r.integers(1, 3)), dilation_w=int(r.integers(0, 3)),
            groups=int(r.choice([1, 1, 2, 3])), direction=int(r.integers(0, 3)),
            mode=int(r.integers(0, 2)), etype=int(r.integers(0, 2)))


def _call(fn):
    try:
        return ("ok", fn())
    except PrimkitError as e:
        return ("err", e.name, str(e))


def test_shape_algebra_matches_reference_sweep(lib, ref):
    for p in _random_problems(3000, 7):
        assert _call(lambda: lib.problem_key(p)) == _call(lambda: ref.problem_key(p))
        assert _call(lambda: lib.output_dims(p)) == _call(lambda: ref.output_dims(p))


def test_solver_registry(lib):
    h = lib.handle()
    assert h.solver_names() == SOLVERS  # exactly 5 built-ins, registry order
    assert h.is_tunable("ImplicitGemm") and not h.is_tunable("Direct")
    with pytest.raises(PrimkitError):
        h.is_tunable("Nope")
    p = problem(n=1, c=4, h=8, w=8, k=4, y=3, x=3, pad=1)
    assert h.is_applicable("Winograd", p)
    p.stride_h = p.stride_w = 2
    assert not h.is_applicable("Winograd", p)
    p = problem(n=1, c=4, h=8, w=8, k=4, y=3, x=3, pad=1)
    assert h.workspace_bytes("Im2colGemm", p) == 4 * 3 * 3 * 8 * 8 * 4  # test_capi.cpp:139-143


def test_solver_queries_match_reference_sweep(lib, ref):
    h, hr = lib.handle(), ref.handle()
    for p in _random_problems(1500, 11):
        for s in SOLVERS:
            assert _call(lambda: h.is_applicable(s, p)) == _call(lambda: hr.is_applicable(s, p))
            assert _call(lambda: h.workspace_bytes(s, p)) == _call(lambda: hr.workspace_bytes(s, p))


def test_run_errors_before_device_work(lib, ref):
    """Solver selection / workspace statuses come first, exactly as in the
    reference (primkit_c.cpp:296-317)."""
    h, hr = lib.handle(), ref.handle()
    p = problem(n=1, c=4, h=8, w=8, k=4, y=3, x=3, pad=1, stride=2)
    a = np.zeros(256, np.float32)
    for solver, ws in (("Winograd", 1 << 30), ("Nope", 0), ("Im2colGemm", 0)):
        got = _call(lambda: h.conv_run(p, solver, a, a, ws))
        want = _call(lambda: hr.conv_run(p, solver, a, a, ws))
        assert got[:2] == want[:2], (solver, got, want)
    pt = problem(n=1, c=4, h=8, w=8, k=4, y=3, x=3, mode=abi.TRANSPOSE,
                 direction=abi.BACKWARD_DATA)
    assert _call(lambda: h.conv_run(pt, None, a, a, 1 << 22))[:2] == ("err", "NO_APPLICABLE_SOLVER")
    assert _call(lambda: h.tune(p, "Direct", 4))[:2] == ("err", "NOT_TUNABLE")


def test_perfdb_roundtrip_and_errors(lib, ref, tmp_path):
    h = lib.handle()
    good = tmp_path / "db.txt"
    good.write_text("# comment\n1-4-6-6-4-3-3-1-1-1-1-1-1-1-F-C-f32=ImplicitGemm:8,8,4;Other:x\n"
                    "0-key=Direct:\n")
    h.perfdb_load(str(good))
    out = tmp_path / "out.txt"
    h.perfdb_save(str(out))
    hr = ref.handle()
    hr.perfdb_load(str(good))
    out_ref = tmp_path / "out_ref.txt"
    hr.perfdb_save(str(out_ref))
    assert out.read_text() == out_ref.read_text()
    assert out.read_text().splitlines()[0] == "0-key=Direct:"
    for bad in ("k=Direct:1\nk=Direct:2\n", "novalue\n", "=x:1\n", "k=\n", "k=;Direct:1\n",
                "k=:1\n"):
        (tmp_path / "bad.txt").write_text(bad)
        got = _call(lambda: h.perfdb_load(str(tmp_path / "bad.txt")))
        want = _call(lambda: hr.perfdb_load(str(tmp_path / "bad.txt")))
        assert got[:2] == want[:2] == ("err", "PARSE_ERROR") and got[2] == want[2], bad
    assert _call(lambda: h.perfdb_load("/nonexistent/none.db"))[1] == "IO_ERROR"


def test_fake_clock_and_counters(lib):
    h = lib.handle()
    h.use_fake_clock()
    t1, t2 = h.now_ms(), h.now_ms()
    assert t2 == t1 + 1.0
    assert h.counters() == (0, 0, 0)


# ---- fusion metadata graph -------------------------------------------------

def _build_plan(L, spec):
    dims, et, conv, ops = spec
    plan = L.fusion_plan(dims, et)
    statuses = []
    if conv is not None:
        fdims, pad, stride, algo = conv
        statuses.append(plan.add_conv(fdims, pad=pad[0], pad_w=pad[1], stride=stride[0],
                                      stride_w=stride[1], algo=algo))
    for op in ops:
        if op[0] == "bias":
            statuses.append(plan.add_bias(op[1]))
        elif op[0] == "bn":
            statuses.append(plan.add_batchnorm(op[1]))
        else:
            statuses.append(plan.add_activation(op[1], 0.1))
    return plan, statuses


def _verdict(L, spec):
    h = L.handle()
    plan, statuses = _build_plan(L, spec)
    if any(statuses):
        return ("add", statuses, L.last_error())
    st = plan.compile(h)
    return ("compile", st, L.last_error() if st else "")


def _fusion_specs(seed, count):
    r = np.random.default_rng(seed)
    algos = ["Direct", "Winograd", "ImplicitGemm", "Im2colGemm", "FFT"]
    for _ in range(count):
        c = int(r.choice([1, 2, 4, 5, 9, 17, 18, 19, 20, 36]))
        k = int(r.integers(1, 9))
        f = int(r.integers(1, 14))
        fx = f if r.random() < 0.9 else int(r.integers(1, 14))
        hw = int(r.integers(max(f, fx), 30))
        pad = (int(r.integers(0, 4)),) * 2 if r.random() < 0.9 else (1, 2)
        stride = (int(r.integers(1, 4)),) * 2 if r.random() < 0.9 else (1, 2)
        et = int(r.integers(0, 2))
        tail = [["bias", k]]
        kind = r.integers(0, 6)
        if kind == 0:
            tail += [["act", int(r.integers(0, 4))]]
        elif kind == 1:
            tail += [["bn", int(r.integers(0, 2))], ["act", int(r.integers(0, 4))]]
        elif kind == 2:
            tail = []
        elif kind == 3:
            tail += [["bn", 1]]
        elif kind == 4:
            tail = [["act", 0], ["bias", k]]
        else:
            tail += [["act", 0], ["act", 1]]
        conv = ((k, c, f, fx), pad, stride, str(r.choice(algos)))
        yield ((1, c, hw, hw), et, conv, tail)
    # norm-activation rows
    for et, mode, act in itertools.product((0, 1), (0, 1), range(4)):
        yield ((2, 3, 4, 4), et, None, [["bn", mode], ["act", act]])
    yield ((2, 3, 4, 4), 0, None, [["bn", 1]])
    yield ((2, 3, 4, 4), 0, None, [["act", 0]])


def test_fusion_verdicts_known_answers(lib):
    # test_capi.cpp:234-251: Winograd 3x3 with c = 17 cites "c >= 18"
    v = _verdict(lib, ((1, 17, 24, 24), 0, ((4, 17, 3, 3), (0, 0), (1, 1), "Winograd"),
                       [["bias", 4], ["act", 0]]))
    assert v[1] == abi.STATUS_CODE["FUSION_NOT_SUPPORTED"] and "c >= 18" in v[2]
    v = _verdict(lib, ((1, 18, 24, 24), 1, ((4, 18, 3, 3), (1, 1), (1, 1), "Winograd"),
                       [["bias", 4], ["act", 0]]))
    assert "bf16" in v[2]
    v = _verdict(lib, ((1, 18, 24, 24), 0, ((4, 18, 3, 3), (1, 1), (1, 1), "ImplicitGemm"),
                       [["bias", 4], ["act", 0]]))
    assert "ImplicitGemm" in v[2]
    v = _verdict(lib, ((1, 18, 24, 24), 0, ((4, 18, 3, 3), (1, 1), (1, 1), "Direct"),
                       [["bias", 4]]))
    assert "prefix" in v[2]
    v = _verdict(lib, ((1, 18, 24, 24), 0, ((4, 18, 3, 3), (0, 0), (1, 1), "Direct"),
                       [["bias", 4], ["bn", 1], ["act", 0]]))
    assert "padding" in v[2]


def test_fusion_verdict_sweep_matches_reference(lib, ref):
    n = 0
    for spec in _fusion_specs(5, 4000):
        assert _verdict(lib, spec) == _verdict(ref, spec), spec
        n += 1
    assert n > 4000


def test_fusion_plan_guards(lib):
    h = lib.handle()
    plan = lib.fusion_plan((2, 4, 6, 6))
    assert plan.add_conv((5, 4, 1, 1)) == 0
    assert plan.add_bias(4) == abi.STATUS_CODE["SHAPE_MISMATCH"]
    assert plan.add_bias(5) == 0
    assert plan.add_activation(abi.LEAKY_RELU, 0.1) == 0
    x = np.zeros((2, 4, 6, 6), np.float32)
    st, _ = plan.execute(h, x, check=False)
    assert st == abi.STATUS_CODE["NOT_COMPILED"]
    assert plan.compile(h) == 0
    assert plan.output_dims() == [2, 5, 6, 6]
    st, _ = plan.execute(h, x, check=False)
    assert st == abi.STATUS_CODE["MISSING_ARGS"]
    assert plan.add_bias(5) == abi.STATUS_CODE["ALREADY_COMPILED"]
