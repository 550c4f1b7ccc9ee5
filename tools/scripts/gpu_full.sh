# full GPU check: tests (+ kernel-variant table), bench line, per-layer report, ncu of the new kernels
set -x
PK_VARIANT_LOG=gpurun_out/variant_coverage.json timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1
tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -c 600 gpurun_out/bench.log
timeout 600 python bench.py --no-extras --steps 10 --layer-report gpurun_out/layers.json > gpurun_out/layers.log 2>&1
head -12 gpurun_out/layers.log
for spec in "conv1 1 stem_dgrad3" "conv1 0 stem_fprop2"; do set -- $spec
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$3 -c 1 -o gpurun_out/ncu_$3 python tools/run_layer.py --layer $1 --dir $2 --iters 1 > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none -k regex:conv_tma_fprop_kernel -c 1 -o gpurun_out/ncu_tf32x3 python tools/bench_configs.py --only cfg1 --iters 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
