mkdir -p gpurun_out/probe
for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_rhopf.so paper_2601_08277_b200/libpicgpu.so build/libpicgpu_rhopf.so; do echo $lib; for o in 3 1 2; do PICGPU_LIB=$lib python tools/jbench.py $o 128 16; done; done > gpurun_out/probe/rho_pf.txt 2>&1
PICGPU_LIB=build/libpicgpu_rhopf.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x -k "rho or density or c2 or C2" 2>&1 | tail -3 >> gpurun_out/probe/rho_pf.txt
