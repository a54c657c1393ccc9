timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/shift_timing.py 0.06 2>&1 | tail -4
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/rc2.json 2>/dev/null
timeout 600 python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/rc4.json 2>/dev/null
timeout 900 python bench.py --config c3o3 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/rc3.json 2>/dev/null
python -c "
import json
for f in ['rc2','rc4','rc3']:
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, '%.3g'%d['value'], round(d['ms_per_step'],3), {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})"
