for L in conv4_2b conv5_2b conv4_1b conv5_1b conv5_1a conv5_2c; do for v in 0 1; do
  PK_WG_PAIR=$v timeout 60 python tools/run_layer.py --layer $L --dir 2 --time 2>&1 | head -1 | sed "s/^/wgpair=$v /"
done; done
