# ncu --set full of the DMMA pencil kernel (J only, C2 QSP) + the fused step kernel
set -x
python tools/jbench.py 3 128 16 > gpurun_out/pp_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_pencil -s 2 -c 1 -o gpurun_out/pp_j python tools/jbench.py 3 128 16 > gpurun_out/pp_ncu.log 2>&1
python bench.py --steps 3 --warmup 3 > gpurun_out/pp_bench_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_pencil -s 3 -c 1 -o gpurun_out/pp_fused python bench.py --steps 3 --warmup 3 > gpurun_out/pp_ncu2.log 2>&1
ls -la gpurun_out
