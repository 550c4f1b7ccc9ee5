for ld in "conv4_2a 0" "conv4_2c 1" "conv5_2a 0" "conv5_2c 0" "conv5_2a 1"; do
  set -- $ld; echo "== $1 dir $2"
  PK_TC2_TRACE=1 timeout 120 python tools/run_layer.py --layer $1 --dir $2 --iters 3 2>&1 | grep tc2
done
