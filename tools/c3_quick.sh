timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --config c3o3 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c3q.json 2>gpurun_out/c3.err || tail -3 gpurun_out/c3.err
PICGPU_FUSE_MAX_MOVED=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c2u.json
python -c "
import json
for f in ['gpurun_out/c3q.json','gpurun_out/c2u.json']:
    d=json.load(open(f)); print(f, round(d['ms_per_step'],3), d['fused_steps'], {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})"
