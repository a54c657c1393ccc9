set -x
mkdir -p gpurun_out/sg
timeout 1500 python -m pytest tests -q -m gpu -x -k "not test_c2_full and not test_c4" 2>&1 | tail -4 > gpurun_out/sg/pytest.log
for r in 1 2; do
timeout 600 python bench.py --config c3o3 --steps 4 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/sg/c3_seg_$r.json 2>&1
PICGPU_PUSH_SEG=0 timeout 600 python bench.py --config c3o3 --steps 4 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/sg/c3_old_$r.json 2>&1
done
PICGPU_FUSE_MAX_MOVED=0 timeout 300 python bench.py --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/sg/c2u_seg.json 2>&1
PICGPU_FUSE_MAX_MOVED=0 PICGPU_PUSH_SEG=0 timeout 300 python bench.py --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/sg/c2u_old.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/sg/launches.csv python bench.py --config c3o3 --steps 2 --warmup 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/sg/ncu.log 2>&1
