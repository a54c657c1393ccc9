mkdir -p gpurun_out/probe
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/probe/c3_launches.csv python bench.py --config c3o3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/probe/c3ncu.log 2>&1
