mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"deposit_current_kernel_v3|k_movers|k_insert|k_borrow" -s 12 -c 4 \
    -o gpurun_out/full_fused python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
