#!/bin/bash
# default-path 128-wide conv_tc layers with the tile-split epilogue (compare profiles/r02_layers.json)
for L in "conv3_1a 0" "conv3_2a 0" "conv3_3a 0" "conv3_2c 1" "conv3_1c 1"; do
  set -- $L
  echo "$1 dir $2: $(timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us') $(timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
done
