for d in 0 1 2 16 3 18 19; do
  PK_STEM_DEBUG=$d timeout 60 python tools/run_layer.py --layer conv1 --dir 2 --time 2>&1 | head -1 | sed "s/^/dbg=$d /"
done
