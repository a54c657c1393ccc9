# radix sort parity + perf, full GPU suite, ncu of the fused kernels at orders 1 and 3
set -x
timeout 900 python -m pytest tests/test_gpu_sort.py -q -x 2>&1 | tail -15 > gpurun_out/s_sort.log
timeout 900 python -m pytest tests -q -m gpu -x -k "not test_c3_geometry and not test_c2_full" 2>&1 | tail -15 > gpurun_out/s_pytest.log
timeout 300 python bench.py --sort resort --steps 5 --no-orders --no-cpu-baseline > gpurun_out/s_resort.json 2>&1
timeout 300 python bench.py --no-orders --no-cpu-baseline --steps 10 > gpurun_out/s_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_v3 -s 3 -c 1 -o gpurun_out/s_fused_o1 python bench.py --order 1 --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/s_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rs_pass -s 0 -c 3 -o gpurun_out/s_rs python bench.py --sort resort --steps 1 --warmup 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/s_ncu2.log 2>&1
