#!/bin/bash
# step A/B of the in-kernel split-K finish cap with the 320-thread wgrad kernel
for i in 1 2 3; do
  for v in 65536 300000 1000000000; do
    echo "fuse_max=$v $(PK_SPLITK_FUSE_MAX=$v timeout 300 python bench.py --no-extras 2>/dev/null | grep -o '"ms_per_step": [0-9.]*')"
  done
done
