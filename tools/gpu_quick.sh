# quick GPU check: tests + C2 bench (+ optional extra bench args in $@)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/qb.json 2> gpurun_out/qb.err; cat gpurun_out/qb.json; tail -5 gpurun_out/qb.err
