# Profiles for profiles/: (1) GPU tests, (2) plain bench run, (3) reference arm,
# (4) launch list of the same bench command (serialised, cold-cache per launch),
# (5) ncu --set full of the fused step kernel, the movers/migration kernels and
# the rho kernel.  Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err || exit 1
cat gpurun_out/prof_bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/prof_ref.json 2> gpurun_out/prof_ref.err; cat gpurun_out/prof_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"deposit_current_kernel_v3" -s 3 -c 1 \
    -o gpurun_out/full_J python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_movers|k_insert|k_borrow" -s 9 -c 3 \
    -o gpurun_out/full_sort python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"density_blocks" -s 2 -c 1 \
    -o gpurun_out/full_rho python tools/jbench.py 3 128 16 > /dev/null 2>&1
for o in 3 2 1; do python tools/jbench.py $o 128 16; done > gpurun_out/jbench.txt
ls -la gpurun_out
