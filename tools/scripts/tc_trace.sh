#!/bin/bash
# PK_TC_TRACE clock stamps of CTA 0 (tile i: 0 producer pre-empty-wait, 1 post, 2/3 MMA tmem_empty wait,
# 4 first full stage, 5/6 epilogue tmem_full wait) for the narrow 1x1 forward
for dbg in 0 7; do
  echo "== conv2_1a fwd PK_TC_DEBUG=$dbg"
  PK_TC_DEBUG=$dbg PK_TC_TRACE=1 timeout 60 python tools/run_layer.py --layer conv2_1a --dir 0 --iters 2 2>&1 | grep "tc tile" | tail -12
done
echo "== conv2_2a fwd (256->64)"
PK_TC_TRACE=1 timeout 60 python tools/run_layer.py --layer conv2_2a --dir 0 --iters 2 2>&1 | grep "tc tile" | tail -12
