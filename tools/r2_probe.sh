# parity of the current tree + ncu (full, source) of the fused QSP kernel
set -x
mkdir -p gpurun_out/probe
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/probe/pytest.log
python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_v3 -s 3 -c 1 -o gpurun_out/probe/fused python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > gpurun_out/probe/ncu.log 2>&1
ncu -i gpurun_out/probe/fused.ncu-rep --page source --csv --print-source sass > gpurun_out/probe/fused_sass.csv 2>/dev/null
ncu -i gpurun_out/probe/fused.ncu-rep --page raw --csv > gpurun_out/probe/fused_raw.csv 2>/dev/null
