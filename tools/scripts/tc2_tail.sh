#!/bin/bash
# gemm_pair_kernel half-tile tail (PK_TC2_TAIL=0: whole tiles only)
for L in "conv5_2a 0" "conv5_2a 1" "conv5_2c 0" "conv5_2c 1" "conv5_1a 0" "conv5_1a 1" "conv4_2a 0" "conv4_2c 1"; do
  set -- $L
  for env in "PK_TC2_TAIL=1" "PK_TC2_TAIL=0"; do
    echo "$1 dir $2 $env: $(env $env timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
  done
done
