PICGPU_J_V4=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_v4m1.so; do
  for v in 0 1; do
    echo -n "$lib v4=$v: "; PICGPU_LIB=$lib PICGPU_J_V4=$v python tools/jbench.py 3 128 16 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('J', round(d['deposit_current_ms'],3))"
    PICGPU_LIB=$lib PICGPU_J_V4=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/v4b.json 2>gpurun_out/v4b.err; python -c "
import json; d=json.load(open('gpurun_out/v4b.json')); print('   step', round(d['ms_per_step'],3), {k:round(v/20,3) for k,v in d['phases_ms_total'].items() if v})" || tail -3 gpurun_out/v4b.err
  done
done
