PK_STEM_TRACE=1 PK_STEM_DEBUG=0 python tools/run_layer.py --layer conv1 --dir 1 --iters 1 2>&1 | tail -12
PK_STEM_TRACE=1 PK_STEM_DEBUG=7 python tools/run_layer.py --layer conv1 --dir 1 --iters 1 2>&1 | tail -12
