# bench lines of every config + slab loopback (NCCL vs torch) + traffic captures
set -x
mkdir -p gpurun_out/b
timeout 600 python bench.py > gpurun_out/b/c2.json 2> gpurun_out/b/c2.err
timeout 300 python bench.py --config c1 --no-orders > gpurun_out/b/c1.json 2> gpurun_out/b/c1.err
timeout 600 python bench.py --config c4 --no-orders > gpurun_out/b/c4.json 2> gpurun_out/b/c4.err
timeout 300 python bench.py --slab --no-orders --no-cpu-baseline > gpurun_out/b/slab_nccl.json 2> gpurun_out/b/slab_nccl.err
timeout 300 python bench.py --slab --exchange torch --no-orders --no-cpu-baseline > gpurun_out/b/slab_torch.json 2> gpurun_out/b/slab_torch.err
timeout 900 python bench.py --config c3o3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/b/c3o3.json 2> gpurun_out/b/c3o3.err
bash tools/traffic.sh
