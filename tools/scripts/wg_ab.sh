#!/bin/bash
# wgrad layer times (one per family instance) + trace of the 256 x 256 drain
for L in conv4_2a conv5_2a conv4_2b conv3_2b conv3_2a conv2_2a conv5_2b conv4_1b conv3_1a; do
  echo "$L $(timeout 60 python tools/run_layer.py --layer $L --dir 2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
done
PK_WG_TRACE=1 timeout 60 python tools/run_layer.py --layer conv5_2a --dir 2 --iters 2 2>&1 | grep "wg:" | tail -1
