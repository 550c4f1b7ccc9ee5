set -x
PK_VARIANT_LOG=gpurun_out/variant_coverage.json timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1
tail -3 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/bench.log 2>&1
tail -c 700 gpurun_out/bench.log
timeout 600 python bench.py --no-extras --steps 10 --layer-report gpurun_out/layers.json > gpurun_out/layers.log 2>&1
head -8 gpurun_out/layers.log
