"""The shipped system perf-db (paper_1910_00078_b200/db/sm100_b200.pkdb, built by
tools/make_perfdb.py on a B200) is a valid reference-format perf-db
(proj/src/core/perfdb.cpp:24-98: "key=solver:values;..." lines) and covers every
problem the benchmark runs: ResNet-50 N=256 forward (ImplicitGemm tile config),
backward data / weights (Im2colGemm#sm100 kernel records) and VGG-16 N=128
forward. Host-only (no GPU): the keys come from the library's problem_key."""
import os

from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import problem
from paper_1910_00078_b200.resnet50 import resnet50_layers, vgg16_layers

DB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                  "paper_1910_00078_b200", "db", "sm100_b200.pkdb")


def _records():
    recs = {}
    for line in open(DB):
        line = line.rstrip("\n")
        if not line or line.startswith("#"):
            continue
        key, rest = line.split("=", 1)
        assert key not in recs
        recs[key] = dict(part.split(":", 1) for part in rest.split(";") if part)
    return recs


def test_shipped_db_covers_the_benchmark(lib):
    recs = _records()
    need = []
    for L in resnet50_layers():
        for d, solver in ((abi.FORWARD, "ImplicitGemm"), (abi.BACKWARD_DATA, "Im2colGemm#sm100"),
                          (abi.BACKWARD_WEIGHTS, "Im2colGemm#sm100")):
            need.append((problem(n=256, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad,
                                 stride=L.stride, direction=d, etype=abi.BF16), solver))
    for L in vgg16_layers():
        need.append((problem(n=128, c=L.c, h=L.h, w=L.h, k=L.k, y=3, x=3, pad=1, etype=abi.BF16),
                     "ImplicitGemm"))
    for p, solver in need:
        key = lib.problem_key(p)
        assert key in recs and solver in recs[key], (key, solver)
        vals = [int(v) for v in recs[key][solver].split(",")]
        if solver == "ImplicitGemm":
            tm, tn, tk = vals  # the reference grid (solver.cpp:185-207)
            assert tm in (1, 2, 4, 8) and tn in (1, 2, 4, 8) and tk in (1, 2, 4)
            assert p.k % tm == 0 and p.c % tk == 0
        else:
            bn, fam, pair, mt, split = vals
            assert bn in (0, 64, 128, 256) and 0 <= fam <= 2 and 0 <= pair <= 2 and 0 <= mt <= 2
            assert 0 <= split <= 16
