set -x
mkdir -p gpurun_out/lp
timeout 1200 python -m pytest tests -q -m gpu -x -k "not test_c3_geometry and not test_c4" 2>&1 | tail -4 > gpurun_out/lp/pytest.log
for r in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/lp/new_$r.json 2>&1
PICGPU_LIB=build/libpicgpu_lp0.so timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/lp/old_$r.json 2>&1
done
for o in 3 2 1; do timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/lp/jbench.log 2>&1; PICGPU_LIB=build/libpicgpu_lp0.so timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/lp/jbench.log 2>&1; done
