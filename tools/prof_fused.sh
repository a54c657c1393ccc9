mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"deposit_current_kernel_v3|k_movers" -s 6 -c 2 \
    -o gpurun_out/full_fused python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
