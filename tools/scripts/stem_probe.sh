for d in 0 1 3 5 7; do PK_STEM_DEBUG=$d python tools/run_layer.py --layer conv1 --dir 2 --time | head -1; done
