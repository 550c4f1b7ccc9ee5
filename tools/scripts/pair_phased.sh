for L in conv3_1b conv4_1b conv5_1b conv3_1ds conv4_1ds conv5_1ds; do for v in 0 1; do
  PK_TMA_PAIR_PHASED=$v timeout 60 python tools/run_layer.py --layer $L --dir 1 --time 2>&1 | head -1 | sed "s/^/pph=$v /"
done; done
timeout 900 python -m pytest tests/test_step_parity_gpu.py tests/test_conv_gpu.py tests/test_large_paths_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
