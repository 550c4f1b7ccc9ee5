python -m pytest tests/test_stem_gpu.py tests/test_conv_bn_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for d in 0 1 2 3 7; do PK_STEM_DEBUG=$d python tools/run_layer.py --layer conv1 --dir 0 --time | head -1; done
