set -x
mkdir -p gpurun_out/ws2
PICGPU_J_WS=1 timeout 900 python -m pytest tests -q -m gpu -x -k "not test_c3_geometry and not test_c4" 2>&1 | tail -5 > gpurun_out/ws2/pytest.log
for o in 3 2 1; do PICGPU_J_WS=1 timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/ws2/jbench.log 2>&1; timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/ws2/jbench.log 2>&1; done
for r in 1 2; do
PICGPU_J_WS=1 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/ws2/b_ws2_$r.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/ws2/b_v3_$r.json 2>&1
done
PICGPU_J_WS=1 PICGPU_LIB=build/libpicgpu_ws1.so timeout 300 python bench.py --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/ws2/b_ws1.json 2>&1
PICGPU_J_WS=1 python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1 && PICGPU_J_WS=1 ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_ws -s 3 -c 1 -o gpurun_out/ws2/ws2_fused python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/ws2/ncu.log 2>&1
