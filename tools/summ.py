import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
for k in ('value', 'ms_per_step', 'gpu_launches', 'phases_ms_total', 'rebuilds', 'moved_fraction', 'clocks'):
    print(k, d.get(k))
r = d['roofline']; print({k: r[k] for k in ('bound', 'frac', 'achieved', 'peak', 'launch_ms', 'deposits_per_s_kernel_only')}); print(r['hbm_view'])
print('e2e', d['e2e'] and d['e2e']['value'], 'cpu', d['cpu_baseline'] and d['cpu_baseline']['value'])
