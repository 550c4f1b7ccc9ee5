for L in conv4_2c conv4_2a conv5_2c; do for n in 8 32 128 256; do python tools/run_layer.py --layer $L --dir 0 --n $n --time | head -1; done; done
