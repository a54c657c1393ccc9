set -x
mkdir -p gpurun_out/probe
for lib in paper_2601_08277_b200/libpicgpu.so build/libpicgpu_l2h2.so; do for r in 1 2; do
  echo "$lib"; for o in 3 1 2; do PICGPU_LIB=$lib python tools/jbench.py $o 128 16; done
done; done > gpurun_out/probe/jonly_l2h.txt 2>&1
