#!/bin/bash
# bench line, per-layer report, step launch list, and a full ncu capture of the narrow 1x1 kernel
timeout 300 python bench.py > gpurun_out/bench_r.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_r2.log 2>&1
timeout 600 python bench.py --layer-report gpurun_out/layers.json > gpurun_out/layers.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/run_step.py > gpurun_out/launches_raw.csv 2> gpurun_out/launches_err.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"conv_tma_wgrad" -s 1 -c 1 -o gpurun_out/r02_wgrad_drain8_conv4_2b python tools/run_layer.py --layer conv4_2b --dir 2 --iters 2 > /dev/null 2>&1
ls gpurun_out
