set -x
mkdir -p gpurun_out/probe
for lib in build/libpicgpu_r0.so paper_2601_08277_b200/libpicgpu.so build/libpicgpu_r0.so paper_2601_08277_b200/libpicgpu.so; do echo $lib; for o in 3 1 2; do PICGPU_LIB=$lib python tools/jbench.py $o 128 16; done; done > gpurun_out/probe/rho_p2.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/probe/pytest.log
