# k_push: spread moved count + wider CTAs; parity + C3 A/B
set -x
mkdir -p gpurun_out/push
timeout 900 python -m pytest tests -q -m gpu -x -k "not test_c2_full and not test_c4" 2>&1 | tail -5 > gpurun_out/push/pytest.log
for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_pn256.so build/libpicgpu_pn1024.so; do
  PICGPU_LIB=$lib timeout 600 python bench.py --config c3o3 --steps 4 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/push/c3_$(basename $lib).json 2>&1
done
python bench.py --config c3o3 --steps 2 --no-orders --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:k_push -s 1 -c 1 -o gpurun_out/push/kpush_c3 python bench.py --config c3o3 --steps 2 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/push/ncu.log 2>&1
