for cfg in "2 0" "2 1" "2 0" "2 1" "1 0"; do set -- $cfg
  extra=""; [ "$2" = "1" ] && extra="--dp"
  timeout 300 python bench.py --no-extras --steps 20 --streams $1 $extra > /tmp/b.json 2>/dev/null
  python - "$1" "$2" <<'PY'
import json, sys
d = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
print("streams", sys.argv[1], "dp", sys.argv[2], round(d["value"], 1), round(d["ms_per_step"], 3), d["clocks"])
PY
done
