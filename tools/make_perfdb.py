"""Build the shipped perf-db (paper_1910_00078_b200/db/sm100_b200.pkdb) on a B200.

For every distinct convolution of the benchmark workloads:
  * ResNet-50 v1.5, 53 conv layers, bf16, N=256 (BASELINE configs[3]/[4], bench.py):
      Forward       ImplicitGemm  primkit_tune (the reference's tile_m/tile_n/tile_k
                                  grid, mapped to the tcgen05 kernel choice)
      BackwardData  Im2colGemm    primkit_tune_kernels ("Im2colGemm#sm100")
      BackwardWeights Im2colGemm  primkit_tune_kernels
  * VGG-16 13 conv layers, bf16, N=128 (BASELINE configs[2]): Forward ImplicitGemm
the tuner times the candidates with CUDA events (1 warm-up + 5 timed, median) on
U(-1,1) device tensors and records the fastest; the db is then the perf-db of
the tuning handle (same text format as the reference's PerfDb, perfdb.cpp:24-98).

    python tools/make_perfdb.py [--out path] [--only resnet,vgg] [--log profiles/r02_tune.jsonl]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1910_00078_b200 import abi  # noqa: E402
from paper_1910_00078_b200.primkit import library, problem  # noqa: E402
from paper_1910_00078_b200.resnet50 import resnet50_layers, vgg16_layers  # noqa: E402

DEFAULT_OUT = os.path.join(ROOT, "paper_1910_00078_b200", "db", "sm100_b200.pkdb")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=DEFAULT_OUT)
    ap.add_argument("--only", default="resnet,vgg")
    ap.add_argument("--log", default=None)
    args = ap.parse_args()
    lib = library()
    h = lib.handle()
    h.load_system_db(None)  # tune from the heuristics, not from a previous db
    log = open(args.log, "w") if args.log else None
    jobs = []
    if "resnet" in args.only:
        for L in resnet50_layers():
            for d in (abi.FORWARD, abi.BACKWARD_DATA, abi.BACKWARD_WEIGHTS):
                jobs.append((f"resnet50/{L.name}", 256, L, d))
    if "vgg" in args.only:
        for L in vgg16_layers():
            jobs.append((f"vgg16/{L.name}", 128, L, abi.FORWARD))
    done = set()
    t0 = time.time()
    for name, n, L, d in jobs:
        p = problem(n=n, c=L.c, h=L.h, w=L.h, k=L.k, y=L.r, x=L.r, pad=L.pad, stride=L.stride,
                    direction=d, etype=abi.BF16)
        key = (lib.problem_key(p), d)
        if key in done:
            continue
        done.add(key)
        rec = {"layer": name, "direction": ["fwd", "bwd_data", "bwd_weights"][d], "key": key[0]}
        if d == abi.FORWARD:
            before = h.kernel_config(p, "ImplicitGemm")
            evals = h.tune(p, "ImplicitGemm", 0, exhaustive=True)
            rec.update(solver="ImplicitGemm", evaluations=evals, default=before,
                       chosen=h.kernel_config(p, "ImplicitGemm"))
        else:
            best, dms, bms = h.tune_kernels(p, "Im2colGemm")
            rec.update(solver="Im2colGemm#sm100", chosen=best, default_ms=dms, best_ms=bms,
                       gain=(dms / bms if bms > 0 else None))
        line = json.dumps(rec)
        print(line, flush=True)
        if log:
            log.write(line + "\n")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    h.perfdb_save(args.out)
    print(json.dumps({"written": args.out, "problems": len(done), "wall_s": time.time() - t0}))


if __name__ == "__main__":
    main()
