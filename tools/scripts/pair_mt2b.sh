for ld in "conv3_1b 0" "conv3_1b 2"; do set -- $ld; for v in 0 1; do
  PK_TMA_PAIR_MT2=$v timeout 60 python tools/run_layer.py --layer $1 --dir $2 --time 2>&1 | head -1 | sed "s/^/pmt2=$v /"
done; done
bash tools/scripts/ab_step.sh PK_TMA_PAIR_MT2
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
