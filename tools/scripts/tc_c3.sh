#!/bin/bash
# conv_tc_kernel<256,6,4> on conv3_2c fwd (128 -> 512 @28): component timing + trace
for dbg in 0 1 4 6 7; do
  echo "PK_TC_DEBUG=$dbg $(PK_TC_DEBUG=$dbg timeout 60 python tools/run_layer.py --layer conv3_2c --dir 0 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
done
PK_TC_TRACE=1 timeout 60 python tools/run_layer.py --layer conv3_2c --dir 0 --iters 2 2>&1 | grep "tc tile" | tail -6
