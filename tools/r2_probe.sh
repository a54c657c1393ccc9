set -x
mkdir -p gpurun_out/probe
( time timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -6 ) > gpurun_out/probe/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/probe/smoke.log 2>&1
( time timeout 900 python bench.py ) > gpurun_out/probe/bench_c2.json 2> gpurun_out/probe/bench_c2.err
