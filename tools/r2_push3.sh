set -x
mkdir -p gpurun_out/p3
timeout 1200 python -m pytest tests -q -m gpu -x -k "not test_c2_full and not test_c4" 2>&1 | tail -5 > gpurun_out/p3/pytest.log
for r in 1 2; do
for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_u1.so build/libpicgpu_u2w.so build/libpicgpu_u2n256.so; do
  PICGPU_LIB=$lib timeout 600 python bench.py --config c3o3 --steps 4 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/p3/c3_$(basename $lib)_$r.json 2>&1
done; done
