#!/bin/bash
# PK_WG_TRACE of CTA (0,0,0): MMA start, last commit, drain start/end, first stage arrivals
for L in conv4_2a conv5_2a conv4_2b conv3_2b conv3_2a; do
  echo "== $L $(timeout 60 python tools/run_layer.py --layer $L --dir 2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
  PK_WG_TRACE=1 timeout 60 python tools/run_layer.py --layer $L --dir 2 --iters 2 2>&1 | grep "wg:" | tail -1
done
