for d in 0 16 4 8; do
echo "== debug $d"
PK_HALO_DEBUG=$d PK_HALO_TRACE=1 timeout 60 python tools/run_layer.py --layer conv2_2b --dir 0 --iters 2 2>&1 | grep "halo tile" | sed -n '10,12p'
PK_HALO_DEBUG=$d timeout 60 python tools/run_layer.py --layer conv2_2b --dir 0 --time | head -1
done
