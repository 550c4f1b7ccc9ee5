for v in 65536 100000000 65536 100000000 65536 100000000; do
  PK_SPLITK_FUSE_MAX=$v timeout 300 python bench.py --no-extras --steps 30 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        b=json.loads(l); print('fuse_max=$v', round(b['ms_per_step'],4), b['clocks']['sm_mhz'])"
done
for L in conv4_2b conv5_2b conv3_2b conv4_2a; do for v in 65536 100000000; do
  PK_SPLITK_FUSE_MAX=$v timeout 60 python tools/run_layer.py --layer $L --dir 2 --time | head -1 | sed "s/^/fm=$v /"
done; done
