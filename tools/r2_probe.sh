set -x
mkdir -p gpurun_out/probe
bash tools/ab_lib.sh paper_2601_08277_b200/libpicgpu.so build/libpicgpu_mb256.so build/libpicgpu_nt128.so build/libpicgpu_mb64.so > gpurun_out/probe/movers_cfg.txt 2>&1
for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_nopf.so; do for r in 1 2; do
  echo "$lib"; PICGPU_LIB=$lib python tools/jbench.py 3 128 16; PICGPU_LIB=$lib python tools/jbench.py 3 128 32
done; done > gpurun_out/probe/jonly_pf.txt 2>&1
