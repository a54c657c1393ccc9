set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -c 3000 gpurun_out/bench_n1.json; tail -5 gpurun_out/bench_n1.err
timeout 300 python bench.py --slab --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_slab1.json 2> gpurun_out/bench_slab1.err; tail -c 1500 gpurun_out/bench_slab1.json; tail -5 gpurun_out/bench_slab1.err
