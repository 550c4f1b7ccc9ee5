#!/bin/bash
# Component timing of conv_tc_kernel on the narrow 1x1 layers (PK_TC_DEBUG bits:
# 1 no MMA, 2 no TMEM load, 4 no store, 8 no math), CUDA-event time per call.
for L in conv2_1a; do
  for D in 0 1; do
    for dbg in 0 1 2 4 6 7; do
      echo "$L dir=$D PK_TC_DEBUG=$dbg: $(PK_TC_DEBUG=$dbg python tools/run_layer.py --layer $L --dir $D --iters 20 --time 2>&1 | grep " us")"
    done
  done
done
