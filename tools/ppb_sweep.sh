timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in ppb1 ppb2 ppb4; do
  echo -n "$v J: "; PICGPU_LIB=build/libpicgpu_$v.so python tools/jbench.py 3 128 16 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['deposit_current_ms'],3))"
  PICGPU_LIB=build/libpicgpu_$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ts.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ts.json')); print('$v step', round(d['ms_per_step'],3), {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})" 2>/dev/null || echo "$v failed"
done
