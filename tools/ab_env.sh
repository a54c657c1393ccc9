# A/B a bench env var: bash tools/ab_env.sh VAR val_a val_b [bench args]
V=$1; A=$2; B=$3; shift 3
for val in $A $B $A $B; do
  env $V=$val timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$V=$val', round(d['ms_per_step'],4), {k:round(v/d['steps'],4) for k,v in d['phases_ms_total'].items() if v})"
done
