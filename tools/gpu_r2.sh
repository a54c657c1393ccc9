set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 > gpurun_out/t1_pytest.log
for o in 3 2 1; do timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/t1_jbench.log 2>&1; PICGPU_J_VARIANT=lane timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/t1_jbench.log 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/t1_bench.json 2> gpurun_out/t1_bench.err
PICGPU_J_VARIANT=lane timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/t1_bench_lane.json 2>> gpurun_out/t1_bench.err
