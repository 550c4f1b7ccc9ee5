#!/bin/bash
# wgrad tile sweep after the 8-warp drain (PK_WG_TILE = NBxMT, PK_WG_PAIR)
for L in conv5_2a conv5_2c conv4_2b conv5_2b conv3_2b conv4_2a conv3_2a; do
  for env in "X=1" "PK_WG_TILE=128x1 PK_WG_PAIR=0" "PK_WG_TILE=128x2 PK_WG_PAIR=0" "PK_WG_TILE=256x1 PK_WG_PAIR=0" "PK_WG_TILE=256x2 PK_WG_PAIR=0" "PK_WG_PAIR=1"; do
    echo "$L $env: $(env $env timeout 60 python tools/run_layer.py --layer $L --dir 2 --iters 3 --time 2>&1 | grep -o '[0-9.]* us')"
  done
done
