# warp-specialised lane kernel: parity, J-only and fused A/B against v3, ncu
set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "not test_c3_geometry and not test_c2_full" 2>&1 | tail -15 > gpurun_out/ws_pytest.log
for o in 3 2 1; do timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/ws_jbench.log 2>&1; PICGPU_J_WS=0 timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/ws_jbench.log 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/ws_bench.json 2> gpurun_out/ws_bench.err
PICGPU_J_WS=0 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/ws_bench_v3.json 2>> gpurun_out/ws_bench.err
ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_ws -s 3 -c 1 -o gpurun_out/ws_fused_o3 python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/ws_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x 2>&1 | tail -5 > gpurun_out/ws_cfg.log
