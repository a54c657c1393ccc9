set -x
mkdir -p gpurun_out/probe
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/probe/pytest.log
for lib in build/libpicgpu_b0.so paper_2601_08277_b200/libpicgpu.so build/libpicgpu_b0.so paper_2601_08277_b200/libpicgpu.so; do
PICGPU_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-orders > gpurun_out/ab.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v}, 'steady', round(d['steady_state']['ms_per_step'],4), round(d['steady_state']['kernel_ms'],4))" >> gpurun_out/probe/borrow.txt
done
