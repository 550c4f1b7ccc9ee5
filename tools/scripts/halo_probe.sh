for d in 0 2 4 6; do PK_HALO_DEBUG=$d python tools/run_layer.py --layer conv2_1b --dir 0 --time | head -1 | sed "s/^/dbg $d /"; done
PK_HALO_TRACE=1 PK_HALO_DEBUG=2 python tools/run_layer.py --layer conv2_1b --dir 0 --iters 1 2>&1 | grep "halo tile" | sed -n 20,24p
