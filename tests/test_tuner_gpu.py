"""The B200 auto-tuner owns real kernel choices:

* the reference's ImplicitGemm grid (tile_m, tile_n, tile_k) maps onto distinct
  tcgen05 kernel instances (a forced family / tile width / CTA-pair choice changes
  the launched template), and every mapped config computes the same convolution;
* primkit_tune_kernels (every direction, any tensor-core solver) records a
  "<solver>#sm100" kernel record that later plans pick up, and the tuned plan's
  output matches the oracle;
* the shipped system perf-db is loaded at handle creation and consulted after
  the user perf-db.
Problems are small (N <= 8) so each direction runs in milliseconds."""
import os

import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(p, seed):
    rng = np.random.default_rng(seed)
    ho = (p.h + 2 * p.pad_h - p.y) // p.stride_h + 1
    x = oracle.round_bf16(rng.uniform(-1, 1, (p.n, p.c, p.h, p.w)).astype(np.float32))
    w = oracle.round_bf16(rng.uniform(-1, 1, (p.k, p.c, p.y, p.x)).astype(np.float32))
    dy = oracle.round_bf16(rng.uniform(-1, 1, (p.n, p.k, ho, ho)).astype(np.float32))
    return x, w, dy


def _run(h, p, solver, x, w, dy):
    if p.direction == abi.FORWARD:
        return h.conv_run(p, solver, x, w), oracle.conv_forward(p, x, w)
    if p.direction == abi.BACKWARD_DATA:
        return h.conv_run(p, solver, dy, w), oracle.conv_backward_data(p, dy, w)
    return h.conv_run(p, solver, dy, x), oracle.conv_backward_weights(p, dy, x)


def test_implicit_gemm_grid_maps_to_distinct_kernels(lib, tmp_path):
    """Different reference tile configs launch different tcgen05 instances on a
    3x3 layer (halo / rectangle / gather; tile widths), all equal to the oracle."""
    h = lib.handle()
    h.load_system_db(None)
    # ResNet-50 conv2_x 3x3 geometry (halo kernel by default)
    p = problem(n=2, c=64, h=56, w=56, k=64, y=3, x=3, pad=1, etype=abi.BF16)
    x, w, dy = _inputs(p, 1)
    variants = {}
    for vals in ("1,1,1", "1,2,1", "1,4,1", "1,2,2", "2,1,1", "1,2,4"):
        path = str(tmp_path / "db.txt")
        with open(path, "w") as f:
            f.write(f"{lib.problem_key(p)}=ImplicitGemm:{vals}\n")
        h.perfdb_load(path)
        got, want = _run(h, p, "ImplicitGemm", x, w, dy)
        assert rel_l2(got, want) <= 1e-2, vals
        variants[vals] = h.last_variant()
    # halo (default), rectangles with two M tiles (tile_n=2), gather (tile_n=4) and
    # rectangles with one M tile (tile_k=2) are four different kernel instances
    assert len({variants[v] for v in ("1,1,1", "1,2,1", "1,4,1", "1,2,2")}) == 4, variants
    assert "halo" in variants["1,1,1"] and "tma" in variants["1,2,1"], variants
    assert "conv_tc_kernel" in variants["1,4,1"], variants


@pytest.mark.parametrize("direction", [abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS])
@pytest.mark.parametrize("shape", [
    dict(n=4, c=64, h=28, w=28, k=256, y=1, x=1),
    dict(n=4, c=128, h=14, w=14, k=128, y=3, x=3, pad=1),
    dict(n=4, c=128, h=28, w=28, k=128, y=3, x=3, pad=1, stride=2),
])
def test_tune_kernels_records_and_plans_use_it(lib, shape, direction):
    h = lib.handle()
    h.load_system_db(None)
    p = problem(**shape, direction=direction, etype=abi.BF16)
    assert h.kernel_config(p, "Im2colGemm") == "0,0,0,0,0"
    best, default_ms, best_ms = h.tune_kernels(p, "Im2colGemm", 64)
    assert 0 < best_ms <= default_ms * 1.02
    assert h.kernel_config(p, "Im2colGemm") == best  # the record is picked up by new plans
    x, w, dy = _inputs(p, 2)
    got, want = _run(h, p, "Im2colGemm", x, w, dy)
    assert rel_l2(got, want) <= 1e-2


def test_forced_choices_compute_the_same_convolution(lib, tmp_path):
    """Every kernel record value set the tuner can emit is a correct convolution."""
    h = lib.handle()
    h.load_system_db(None)
    cases = [
        (dict(n=4, c=256, h=14, w=14, k=256, y=3, x=3, pad=1), abi.FORWARD, "ImplicitGemm"),
        (dict(n=4, c=256, h=14, w=14, k=512, y=1, x=1), abi.BACKWARD_DATA, "Im2colGemm"),
        (dict(n=4, c=256, h=14, w=14, k=256, y=3, x=3, pad=1), abi.BACKWARD_WEIGHTS, "Im2colGemm"),
    ]
    records = ["0,0,0,0,0", "128,0,0,0,0", "64,1,1,1,0", "0,2,0,0,0", "0,0,2,2,0", "256,1,2,0,8",
               "128,0,1,2,2", "0,1,0,1,0"]
    for shape, d, solver in cases:
        p = problem(**shape, direction=d, etype=abi.BF16)
        x, w, dy = _inputs(p, 3)
        for r in records:
            db = tmp_path / "k.txt"
            db.write_text(f"{lib.problem_key(p)}={solver}#sm100:{r}\n")
            h.perfdb_load(str(db))
            assert h.kernel_config(p, solver) == r
            got, want = _run(h, p, solver, x, w, dy)
            assert rel_l2(got, want) <= 1e-2, (shape, d, r, h.last_variant())


def test_system_db_loaded_and_consulted_after_user_db(lib, tmp_path):
    h = lib.handle()
    path, n = h.system_db()
    shipped = os.path.join(ROOT, "paper_1910_00078_b200", "db", "sm100_b200.pkdb")
    if os.path.exists(shipped):
        assert os.path.samefile(path, shipped) and n > 0
    p = problem(n=2, c=64, h=8, w=8, k=64, y=3, x=3, pad=1, direction=abi.BACKWARD_DATA,
                etype=abi.BF16)
    sysdb = tmp_path / "sys.pkdb"
    sysdb.write_text(f"{lib.problem_key(p)}=Im2colGemm#sm100:128,1,0,0,0\n")
    h.load_system_db(str(sysdb))
    assert h.system_db() == (str(sysdb), 1)
    assert h.kernel_config(p, "Im2colGemm") == "128,1,0,0,0"
    user = tmp_path / "user.txt"
    user.write_text(f"{lib.problem_key(p)}=Im2colGemm#sm100:64,0,0,0,0\n")
    h.perfdb_load(str(user))
    assert h.kernel_config(p, "Im2colGemm") == "64,0,0,0,0"  # the user record wins
    h.load_system_db(None)
    assert h.system_db() == ("", 0)
