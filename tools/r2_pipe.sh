set -x
mkdir -p gpurun_out/pp
timeout 1200 python -m pytest tests -q -m gpu -x -k "not test_c2_full and not test_c4" 2>&1 | tail -4 > gpurun_out/pp/pytest.log
for r in 1 2; do
timeout 600 python bench.py --config c3o3 --steps 4 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/pp/c3_pipe256_$r.json 2>&1
PICGPU_PUSH_PIPE=0 timeout 600 python bench.py --config c3o3 --steps 4 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/pp/c3_old_$r.json 2>&1
done
PICGPU_LIB=build/libpicgpu_pp512.so timeout 600 python bench.py --config c3o3 --steps 4 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/pp/c3_pipe512.json 2>&1
PICGPU_LIB=build/libpicgpu_pp128.so timeout 600 python bench.py --config c3o3 --steps 4 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/pp/c3_pipe128.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_push -c 3 --csv --log-file gpurun_out/pp/kpush.csv python bench.py --config c3o3 --steps 2 --warmup 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/pp/ncu.log 2>&1
