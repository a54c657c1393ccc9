# A/B two libraries on the C2 bench: bash tools/ab_lib.sh libA libB
for r in 1 2; do for lib in "$@"; do
  PICGPU_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})" 2>/dev/null || echo "$lib failed"
done; done
