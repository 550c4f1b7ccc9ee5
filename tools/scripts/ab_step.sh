# A/B of one env knob on the whole bench step (same box, alternating)
KNOB=${1:-PK_HALO_MT2}
for v in 0 1 0 1 0 1; do
  env $KNOB=$v timeout 300 python bench.py --no-extras --steps 30 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        b=json.loads(l); print('$KNOB=$v', round(b['ms_per_step'],4), b['clocks']['sm_mhz'])"
done
