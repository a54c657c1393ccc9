# fused vs unfused step on the other configs: bash tools/cfg_sweep.sh cfg...
for cfg in "$@"; do for f in 1 0; do
  PICGPU_FUSE_MAX_MOVED=$f timeout 600 python bench.py --config $cfg --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cs.json 2>gpurun_out/cs.err || tail -3 gpurun_out/cs.err
  python -c "
import json; d=json.load(open('gpurun_out/cs.json')); print('$cfg fused=$f', '%.3g'%d['value'], round(d['ms_per_step'],3), 'moved', round(d['moved_fraction'],4), 'rebuilds', d['rebuilds'], {k:round(v/d['steps'],3) for k,v in d['phases_ms_total'].items() if v})"
done; done
