set -x
mkdir -p gpurun_out/probe
for lib in build/libpicgpu_rl2.so paper_2601_08277_b200/libpicgpu.so; do
PICGPU_LIB=$lib timeout 900 python bench.py --config c3o3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib c3o3', round(d['ms_per_step'],3), d['rebuilds'], {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})" >> gpurun_out/probe/relayout.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_relayout_fill -c 2 --csv --log-file gpurun_out/probe/rl_c4.csv python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/probe/pytest.log
