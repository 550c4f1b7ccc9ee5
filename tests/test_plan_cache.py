"""Plan cache levels through the C ABI — the reference's test_tuning.cpp:242-299
("plan cache: memory, disk and corruption levels", "plan cache degrades to
memory-only on unwritable dir") restated. primkit_conv_device_workspace makes
exactly one cached_build per call and touches no device, so the levels are
checked on CPU; the GPU half (a disk-hit plan runs bit-identically to a fresh
build) is test_plan_cache_disk_hit_runs_identically."""
import os

import numpy as np
import pytest

from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem


def tunable_problem():
    # reference tests/test_tuning.cpp tunable_problem(): small 3x3 forward
    return problem(n=1, c=4, h=6, w=6, k=4, y=3, x=3, pad=1)


def test_memory_disk_and_corruption_levels(lib, tmp_path):
    d = str(tmp_path / "cache")
    p = tunable_problem()
    with lib.handle() as h:
        h.set_cache_dir(d)
        h.device_workspace(p, "Im2colGemm")
        assert h.plan_cache_stats() == (1, 0, 0)
        h.device_workspace(p, "Im2colGemm")
        assert h.plan_cache_stats() == (1, 1, 0)
    files = os.listdir(d)
    assert len(files) == 1 and files[0].endswith(".plan")
    body = open(os.path.join(d, files[0])).read()
    assert body.startswith("primkit-plan v1\n")
    with lib.handle() as h:  # fresh handle over the same directory: disk hit, no build
        h.set_cache_dir(d)
        h.device_workspace(p, "Im2colGemm")
        assert h.plan_cache_stats() == (0, 0, 1)
    for f in os.listdir(d):  # corrupt every entry: the next build silently rebuilds
        with open(os.path.join(d, f), "w") as fh:
            fh.write("garbage")
    with lib.handle() as h:
        h.set_cache_dir(d)
        h.device_workspace(p, "Im2colGemm")
        assert h.plan_cache_stats() == (1, 0, 0)
    assert open(os.path.join(d, files[0])).read() == body  # rewritten


def test_distinct_solvers_and_problems_get_distinct_entries(lib, tmp_path):
    d = str(tmp_path / "c2")
    with lib.handle() as h:
        h.set_cache_dir(d)
        p = tunable_problem()
        for s in ("Im2colGemm", "Direct", "ImplicitGemm"):
            h.device_workspace(p, s)
        q = problem(n=2, c=4, h=6, w=6, k=4, y=3, x=3, pad=1)
        h.device_workspace(q, "Direct")
        assert h.plan_cache_stats() == (4, 0, 0)
    assert len(os.listdir(d)) == 4


def test_unwritable_dir_degrades_to_memory_only(lib):
    with lib.handle() as h:
        h.set_cache_dir("/proc/definitely/not/writable")
        p = tunable_problem()
        h.device_workspace(p, "Direct")
        h.device_workspace(p, "Direct")
        assert h.plan_cache_stats() == (1, 1, 0)


@pytest.mark.gpu
def test_plan_cache_disk_hit_runs_identically(lib, tmp_path):
    """Cached (disk-hit) and freshly built plans produce bit-identical
    results (test_tuning.cpp:269-271)."""
    d = str(tmp_path / "c3")
    p = problem(n=2, c=64, h=14, w=14, k=64, y=3, x=3, pad=1, etype=abi.BF16)
    sa, sb, _ = operand_shapes(lib, p)
    rng = np.random.default_rng(55)
    a = rng.uniform(-1, 1, sa).astype(np.float32)
    b = rng.uniform(-1, 1, sb).astype(np.float32)
    with lib.handle() as h:
        h.set_cache_dir(d)
        r1 = h.conv_run(p, "ImplicitGemm", a, b)
        assert h.plan_cache_stats()[0] == 1
    with lib.handle() as h:
        h.set_cache_dir(d)
        r2 = h.conv_run(p, "ImplicitGemm", a, b)
        assert h.plan_cache_stats() == (0, 0, 1)
    assert np.array_equal(r1, r2)
