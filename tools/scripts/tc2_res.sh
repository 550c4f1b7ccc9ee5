#!/bin/bash
# resident-filter-half pair GEMM (reduction 256) vs the single-CTA PLAIN_RES_BIG (PK_TC2_RES=0)
for L in "conv4_2c 0" "conv4_2a 1" "conv4_1a 1" "conv4_1c 0"; do
  set -- $L
  for env in "PK_TC2_RES=1" "PK_TC2_RES=0"; do
    echo "$1 dir $2 $env: $(env $env timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
  done
done
PK_TC2_TRACE=1 timeout 60 python tools/run_layer.py --layer conv4_2c --dir 0 --iters 2 2>&1 | grep "tc2:" | tail -1
