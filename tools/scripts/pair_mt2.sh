for L in conv3_2b conv3_3b; do for d in 0 1; do for v in 0 1 0 1; do
  PK_TMA_PAIR_MT2=$v timeout 60 python tools/run_layer.py --layer $L --dir $d --time 2>&1 | head -1 | sed "s/^/pmt2=$v /"
done; done; done
PK_TMA_PAIR_MT2=1 timeout 900 python -m pytest tests/test_step_parity_gpu.py tests/test_conv_gpu.py tests/test_large_paths_gpu.py tests/test_fusion_bn_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
