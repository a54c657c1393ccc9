set -x
mkdir -p gpurun_out/sl
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_dropin.py tests/test_gpu_parity.py -q -x 2>&1 | tail -4 > gpurun_out/sl/pytest.log
for r in 1 2; do timeout 300 python bench.py --slab --no-orders --no-cpu-baseline > gpurun_out/sl/slab_$r.json 2>&1; done
