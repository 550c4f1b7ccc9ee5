python -m pytest tests/test_halo_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in 1 0; do for L in conv3_2b; do for d in 0 1; do PK_HALO_MT2=$v python tools/run_layer.py --layer $L --dir $d --time | head -1 | sed "s/^/mt2=$v /"; done; done; done
python tools/run_layer.py --layer conv2_1b --dir 0 --time | head -1
