#!/bin/bash
# conv_tc_kernel epilogue: TMA store vs coalesced st.global from the staging (PK_TC_STORE=1)
for L in "conv3_2c 0" "conv3_2a 1" "conv2_2c 0" "conv2_1a 0" "conv4_2c 0" "conv3_1c 0"; do
  set -- $L
  for env in "PK_TC_STORE=0" "PK_TC_STORE=1"; do
    echo "$1 dir $2 $env: $(env $env timeout 60 python tools/run_layer.py --layer $1 --dir $2 --iters 5 --time 2>&1 | grep -o '[0-9.]* us')"
  done
done
