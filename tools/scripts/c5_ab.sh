#!/bin/bash
# conv5 1x1 layers (M = 12544 rows): tile width A/B (wave quantization of 256-wide pair tiles)
for L in "conv5_2a 0" "conv5_2a 1" "conv5_2c 0" "conv5_2c 1" "conv5_1a 0" "conv4_2a 0"; do
  set -- $L
  for env in "X=1" "PK_TC_BN=128" "PK_TC2_ALL=1" "PK_TC_BN=64"; do
    echo "$1 dir $2 $env: $(env $env timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
  done
done
PK_TC2_TRACE=1 timeout 60 python tools/run_layer.py --layer conv5_2a --dir 0 --iters 2 2>&1 | grep -v "^done" | tail -12
