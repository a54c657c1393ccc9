mkdir -p gpurun_out/probe
for r in 1 2; do for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_cicpf.so; do
  PICGPU_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-orders --steady-steps 0 --order 1 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib c2 order 1', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})"
  PICGPU_LIB=$lib timeout 300 python bench.py --config c1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-orders --steady-steps 0 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib c1', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})"
done; done > gpurun_out/probe/cicpf.txt 2>&1
