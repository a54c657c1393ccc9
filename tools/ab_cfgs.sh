# A/B libraries over the C2 box at orders 3/1/2 and C1: bash tools/ab_cfgs.sh libA libB ...
for r in 1 2; do for lib in "$@"; do
  for o in 3 1 2; do
    PICGPU_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-orders --steady-steps 0 --order $o > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib c2 order $o', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})"
  done
  PICGPU_LIB=$lib timeout 300 python bench.py --config c1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-orders --steady-steps 0 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib c1', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})"
done; done
