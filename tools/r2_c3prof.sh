set -x
mkdir -p gpurun_out/c3p
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/c3p/launches.csv python bench.py --config c3o3 --steps 5 --warmup 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/c3p/ncu.log 2>&1
timeout 600 python bench.py --config c3o3 --steps 5 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/c3p/bench.json 2>&1
