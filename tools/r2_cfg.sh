# full-size config parity + the new bench line (orders, one-core CPU arm)
set -x
timeout 1500 python -m pytest tests/test_gpu_configs.py -v -x --durations=0 2>&1 | tail -30 > gpurun_out/cfg_pytest.log
timeout 600 python bench.py > gpurun_out/cfg_bench.json 2> gpurun_out/cfg_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/cfg_ref.json 2> gpurun_out/cfg_ref.err
