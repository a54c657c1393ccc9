for v in p8x4 p16x2 p4x8 p8x2m4 p16x4m2; do
  PICGPU_LIB=build/libpicgpu_$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ts.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ts.json')); print('$v', round(d['ms_per_step'],3), {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})" 2>/dev/null || echo "$v failed"
done
