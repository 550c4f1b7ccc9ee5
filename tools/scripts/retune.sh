# re-tune the shipped perf-db with this tree's kernels, then A/B the bench step against the old db
timeout 2400 python tools/make_perfdb.py --out gpurun_out/new.pkdb --log gpurun_out/tune_new.jsonl > gpurun_out/tune_stdout.txt 2>&1
tail -1 gpurun_out/tune_stdout.txt
for i in 1 2 3; do
  for db in paper_1910_00078_b200/db/sm100_b200.pkdb gpurun_out/new.pkdb; do
    PRIMKIT_SYSTEM_DB=$db timeout 300 python bench.py --no-extras --steps 30 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        b=json.loads(l); print('$db', round(b['ms_per_step'],4), b['clocks']['sm_mhz'])"
  done
done
