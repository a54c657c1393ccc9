# sorter change check: GPU parity of the sort paths + C2/C3/C4 step timings
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4

timeout 300 python tools/c3_sort_prof.py 2>&1 | tail -4
for c in c2 c3o3 c4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$c', d['value'], d['ms_per_step'], {k: round(v/10,3) for k,v in d['config'].get('phases_ms_total',d.get('phases_ms_total',{})).items()}, d['roofline']['frac'])"
done
