for ld in "conv5_2a 0" "conv5_2a 1" "conv5_2c 0" "conv5_2c 1" "conv4_2a 0"; do
  set -- $ld
  for env in "X=1" "PK_TC_BN=128" "PK_TC2=0" "PK_TC_BN=128 PK_TC2=0"; do
    echo -n "$env  "; env $env timeout 120 python tools/run_layer.py --layer $1 --dir $2 --time | head -1
  done
done
