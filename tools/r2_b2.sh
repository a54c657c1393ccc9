set -x
mkdir -p gpurun_out/b2
timeout 600 python -m pytest tests/test_gpu_lwfa.py tests/test_gpu_dropin.py -q -x 2>&1 | tail -8 > gpurun_out/b2/pytest.log
timeout 600 python bench.py --config c4 --no-orders --no-cpu-baseline > gpurun_out/b2/c4.json 2> gpurun_out/b2/c4.err
timeout 300 python bench.py --slab --no-orders --no-cpu-baseline > gpurun_out/b2/slab_nccl.json 2> gpurun_out/b2/slab_nccl.err
timeout 300 python bench.py --slab --exchange torch --no-orders --no-cpu-baseline > gpurun_out/b2/slab_torch.json 2> gpurun_out/b2/slab_torch.err
