for d in 0 32; do for dir in 0 1; do PK_HALO_DEBUG=$d python tools/run_layer.py --layer conv2_1b --dir $dir --time | head -1 | sed "s/^/dbg $d /"; done; done
