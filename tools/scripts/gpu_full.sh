# full GPU check: tests (+ kernel-variant table), bench line, per-layer report
set -x
PK_VARIANT_LOG=gpurun_out/variant_coverage.json timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1
tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -c 1500 gpurun_out/bench.log
timeout 600 python bench.py --no-extras --steps 10 --layer-report gpurun_out/layers.json > gpurun_out/layers.log 2>&1
head -30 gpurun_out/layers.log
