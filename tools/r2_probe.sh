mkdir -p gpurun_out/probe
for c in c3o1 c3o2; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/probe/bench_$c.json 2> gpurun_out/probe/bench_$c.err; done
