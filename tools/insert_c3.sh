# k_insert grid multiplier at C3 (runtime env): bash tools/insert_c3.sh 4 8 16
for m in "$@"; do
  PICGPU_INSERT_BLOCKS=$m timeout 900 python bench.py --config c3o3 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ins.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ins.json')); print('mult $m c3', round(d['ms_per_step'],3), {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})" || echo "$m failed"
  PICGPU_INSERT_BLOCKS=$m timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ins2.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ins2.json')); print('mult $m c2', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})" || echo "$m failed"
done
