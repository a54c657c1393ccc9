# round-2 state check on one B200: GPU tests, C2 bench, smoke
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 > gpurun_out/r2_pytest.log
timeout 300 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
for o in 3 2 1; do timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/r2_jbench.log 2>&1; done
