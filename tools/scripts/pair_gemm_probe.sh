# gemm_pair_kernel layers: timing (graph of 10 calls) + parity of the large paths
for ld in "conv4_2a 0" "conv4_2c 1" "conv5_2a 0" "conv5_2c 1" "conv4_1c 1" "conv5_1a 0"; do
  set -- $ld; timeout 120 python tools/run_layer.py --layer $1 --dir $2 --time | head -1
done
timeout 900 python -m pytest tests/test_large_paths_gpu.py tests/test_step_parity_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
