mkdir -p gpurun_out/probe
bash tools/ab_cfgs.sh paper_2601_08277_b200/libpicgpu.so build/libpicgpu_zw2.so build/libpicgpu_zw6.so build/libpicgpu_zw8.so > gpurun_out/probe/zw.txt 2>&1
