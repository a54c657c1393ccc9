# final validation of the tree: GPU suite, smoke, default bench (timed), reference arm, MINB A/B
set -x
mkdir -p gpurun_out/f1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f1/smi.txt
( time timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -8 ) > gpurun_out/f1/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1/smoke.log 2>&1
( time timeout 900 python bench.py ) > gpurun_out/f1/bench.json 2> gpurun_out/f1/bench.err
for r in 1 2; do PICGPU_LIB=build/libpicgpu_lm2.so timeout 300 python bench.py --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/f1/lm2_$r.json 2>&1; done
python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f1/launches.csv python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/f1/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_v3 -s 3 -c 1 -o gpurun_out/f1/fused_v3 python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/f1/ncu_f.log 2>&1
