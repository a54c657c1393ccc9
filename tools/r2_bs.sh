set -x
mkdir -p gpurun_out/bs
timeout 1200 python -m pytest tests -q -m gpu -x -k "not test_c3_geometry and not test_c4" 2>&1 | tail -4 > gpurun_out/bs/pytest.log
PICGPU_J_WS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" 2>&1 | tail -3 > gpurun_out/bs/pytest_ws.log
for r in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bs/new_$r.json 2>&1
PICGPU_LIB=build/libpicgpu_bs0.so timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bs/old_$r.json 2>&1
done
for o in 3 2 1; do timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/bs/jbench.log 2>&1; PICGPU_LIB=build/libpicgpu_bs0.so timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/bs/jbench.log 2>&1; done
PICGPU_J_WS=1 timeout 300 python bench.py --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/bs/ws_new.json 2>&1
