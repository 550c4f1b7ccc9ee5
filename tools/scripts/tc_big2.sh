#!/bin/bash
# PLAIN_RES_BIG (conv4 1x1) layers after the direct-store / 6-stage change
for L in conv4_2c conv4_1c conv4_2a; do for D in 0 1; do
  timeout 60 python tools/run_layer.py --layer $L --dir $D --iters 5 --time 2>&1 | grep " us"
done; done
for L in conv3_1a conv3_2a conv5_2a conv2_1a; do for D in 0 1; do
  timeout 60 python tools/run_layer.py --layer $L --dir $D --iters 5 --time 2>&1 | grep " us"
done; done
PK_TC_TRACE=1 timeout 60 python tools/run_layer.py --layer conv4_2c --dir 0 --iters 2 2>&1 | grep "tc tile" | tail -6
