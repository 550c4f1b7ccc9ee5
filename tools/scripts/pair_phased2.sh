bash tools/scripts/ab_step.sh PK_TMA_PAIR_PHASED
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
