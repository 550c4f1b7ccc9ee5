#!/bin/bash
# tile-split epilogue for 128-wide tiles (4 TMEM buffers) vs the 256-wide default
for L in "conv3_2c 0" "conv3_2a 1" "conv2_2c 0" "conv3_1a 0" "conv4_2c 0" "conv2_1a 0"; do
  set -- $L
  for env in "X=1" "PK_TC_BN=128"; do
    echo "$1 dir $2 $env: $(env $env timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
  done
done
