# two-phase k_movers: parity suites, A/B on C2 (orders 3, 1, 2), C4 quick
set -x
mkdir -p gpurun_out/probe
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/probe/pytest.log
bash tools/ab_lib.sh build/libpicgpu_base.so paper_2601_08277_b200/libpicgpu.so > gpurun_out/probe/ab.txt 2>&1
for lib in build/libpicgpu_base.so paper_2601_08277_b200/libpicgpu.so; do
  for o in 1 2; do
  PICGPU_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-orders --order $o > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib order $o', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})" >> gpurun_out/probe/ab.txt
  done
  PICGPU_LIB=$lib timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib c4', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})" >> gpurun_out/probe/ab.txt
done
