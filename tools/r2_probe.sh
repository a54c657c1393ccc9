set -x
mkdir -p gpurun_out/probe
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/probe/pytest.log
timeout 600 python bench.py > gpurun_out/probe/bench_c2.json 2> gpurun_out/probe/bench_c2.err
for o in 3 2 1; do python tools/jbench.py $o 128 16; done > gpurun_out/probe/jbench.txt 2>&1
