# C3 crossover: incremental sort vs full re-sort every step, orders 1/2/3 (BASELINE configs[2])
mkdir -p gpurun_out
for cfg in c3o1 c3o2 c3o3; do for srt in incremental resort; do
  timeout 900 python bench.py --config $cfg --sort $srt --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_${cfg}_${srt}.json 2>gpurun_out/c3.err || tail -3 gpurun_out/c3.err
  python -c "
import json; d=json.load(open('gpurun_out/c3_${cfg}_${srt}.json')); print('$cfg $srt', '%.3g'%d['value'], round(d['ms_per_step'],2), 'moved', round(d['moved_fraction'],4), 'fused', d.get('fused_steps'), 'rebuilds', d['rebuilds'], {k:round(v/d['steps'],2) for k,v in d['phases_ms_total'].items() if v}, 'roof', round(d['roofline']['frac'],3))"
done; done
