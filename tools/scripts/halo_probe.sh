python -m pytest tests/test_halo_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for rt in 1 0; do for L in conv2_1b; do for d in 0 1; do PK_HALO_ROWTILE=$rt python tools/run_layer.py --layer $L --dir $d --time | head -1 | sed "s/^/rowtile $rt /"; done; done; done
PK_HALO_TRACE=1 python tools/run_layer.py --layer conv2_1b --dir 0 --iters 1 2>&1 | grep "halo tile" | sed -n 20,24p
