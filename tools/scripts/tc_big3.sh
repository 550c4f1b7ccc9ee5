#!/bin/bash
# conv4 1x1 256->1024 (fwd of conv4_xc, dgrad of conv4_xa): resident-B big vs pair GEMM vs 128-wide tiles
for L in "conv4_2c 0" "conv4_2a 1" "conv5_2c 0" "conv3_2c 0"; do
  set -- $L
  echo "$1 dir $2 default: $(timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
  echo "$1 dir $2 PK_TC2_ALL: $(PK_TC2_ALL=1 timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
  echo "$1 dir $2 PK_TC_BN=128: $(PK_TC_BN=128 timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
done
