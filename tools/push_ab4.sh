# A/B k_push variants at C3 (unfused high-migration step) and C2 unfused: bash tools/push_ab4.sh libA libB ...
for lib in "$@"; do
  PICGPU_LIB=$lib timeout 900 python bench.py --config c3o3 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pa3.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pa3.json')); print('$lib c3', round(d['ms_per_step'],3), {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})" || echo "$lib c3 failed"
  PICGPU_LIB=$lib PICGPU_FUSE_MAX_MOVED=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pa.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pa.json')); print('$lib c2u', round(d['ms_per_step'],3), {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})" || echo "$lib c2 failed"
done
