set -x
mkdir -p gpurun_out/f2
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/f2/pytest.log
( time timeout 900 python bench.py ) > gpurun_out/f2/bench.json 2> gpurun_out/f2/bench.err
