#!/bin/bash
# narrow (BN=64) conv_tc layers: CUDA-event time per call, then the trace
for L in conv2_1a conv2_2a; do for D in 0 1; do
  timeout 60 python tools/run_layer.py --layer $L --dir $D --iters 5 --time 2>&1 | grep " us"
done; done
timeout 60 python tools/run_layer.py --layer conv2_1c --dir 1 --iters 5 --time 2>&1 | grep " us"
PK_TC_TRACE=1 timeout 60 python tools/run_layer.py --layer conv2_1a --dir 0 --iters 2 2>&1 | grep "tc tile" | tail -6
