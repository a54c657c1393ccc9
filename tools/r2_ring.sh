# per-lane cp.async record ring (CIC fused pass): parity + A/B
set -x
mkdir -p gpurun_out/ring
timeout 900 python -m pytest tests -q -m gpu -x -k "not test_c3_geometry and not test_c2_full and not test_c4" 2>&1 | tail -5 > gpurun_out/ring/pytest.log
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "c1 or c3_geometry and 1" 2>&1 | tail -5 > gpurun_out/ring/cfg.log
for r in 1 2; do
for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_cr0.so build/libpicgpu_cr3.so; do
  PICGPU_LIB=$lib timeout 300 python bench.py --order 1 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/ring/o1_$(basename $lib)_$r.json 2>&1
done
for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_qr3.so; do
  PICGPU_LIB=$lib timeout 300 python bench.py --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/ring/o3_$(basename $lib)_$r.json 2>&1
done
done
python bench.py --order 1 --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_v3 -s 3 -c 1 -o gpurun_out/ring/cic_ring python bench.py --order 1 --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/ring/ncu.log 2>&1
