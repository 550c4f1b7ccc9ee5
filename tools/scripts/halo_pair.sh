for v in "PK_HALO_MT2=0" "X=1" "PK_HALO_PAIR=1" "PK_HALO_MT2=0" "X=1"; do
 env $v timeout 60 python tools/run_layer.py --layer conv2_2b --dir 0 --time 2>&1 | head -1 | sed "s/^/$v /"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
