for d in 32 0; do
for ld in "conv2_2b 0" "conv2_2b 1" "conv3_2b 0"; do set -- $ld
PK_HALO_DEBUG=$d timeout 60 python tools/run_layer.py --layer $1 --dir $2 --time | head -1 | sed "s/^/dbg=$d /"
done; done
PK_HALO_TRACE=1 timeout 60 python tools/run_layer.py --layer conv2_2b --dir 0 --iters 2 2>&1 | grep "halo tile" | sed -n '10,13p'
timeout 900 python -m pytest tests/test_halo_gpu.py tests/test_step_parity_gpu.py tests/test_fusion_bn_gpu.py tests/test_conv_bn_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
