for L in conv4_2b conv5_2b conv4_1ds conv3_1ds conv5_1ds conv4_1b conv5_1b; do for v in 0 1; do
  PK_TMA_PAIR=$v PK_VARIANT_LOG=gpurun_out/v_$L_$v.json timeout 60 python tools/run_layer.py --layer $L --dir 0 --time 2>&1 | head -1 | sed "s/^/pair=$v /"
done; done
