for bn in 0 128; do for L in conv4_1b conv5_1b conv4_1ds conv5_1ds conv3_1ds; do PK_TMA_BN=$bn python tools/run_layer.py --layer $L --dir 1 --time | head -1 | sed "s/^/bn=$bn /"; done; done
