# C3 (256^3 x 32 ppc, 11% movers per step): unfused (default above 6%) vs fused step
for f in 0 1; do
  PICGPU_FUSE_MAX_MOVED=$f timeout 900 python bench.py --config c3o3 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c3f.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c3f.json')); print('c3 fuse=$f', round(d['ms_per_step'],3), d['fused_steps'], d['rebuilds'], {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})"
done
