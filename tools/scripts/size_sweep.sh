# time vs batch size: fixed per-launch overhead = intercept of t(N)
for ld in "conv4_2a 0" "conv4_2a 1" "conv4_2a 2" "conv4_2c 0" "conv5_2a 0" "conv2_2a 0" "conv3_2b 0"; do
  set -- $ld
  for n in 32 64 128 256 512; do timeout 120 python tools/run_layer.py --layer $1 --dir $2 --n $n --time | head -1; done
done
