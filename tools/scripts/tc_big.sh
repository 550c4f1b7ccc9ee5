#!/bin/bash
# conv_tc_kernel PLAIN_RES_BIG (conv4 1x1 256 -> 1024): component timing + trace
for dbg in 0 1 2 4 8 14; do
  echo "PK_TC_DEBUG=$dbg $(PK_TC_DEBUG=$dbg timeout 60 python tools/run_layer.py --layer conv4_2c --dir 0 --iters 5 --time 2>&1 | grep ' us')"
done
PK_TC_TRACE=1 timeout 60 python tools/run_layer.py --layer conv4_2c --dir 0 --iters 2 2>&1 | grep "tc tile" | tail -8
