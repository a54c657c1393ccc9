# Final-tree validation and profiles (r02, end): GPU suite, smoke, default bench (timed), reference arm, launch list,
# ncu --set full of the fused kernels (QSP, CIC), C1/C4/C3/slab bench lines, DRAM traffic of the C2/C1/C4 kernels.
set -x
O=gpurun_out/f4
mkdir -p $O gpurun_out/traffic
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
( time timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -8 ) > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time timeout 900 python bench.py ) > $O/bench_c2.json 2> $O/bench_c2.err
( time timeout 900 python bench.py --impl reference ) > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 20 --warmup 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > $O/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_v3 -s 3 -c 1 -o $O/fused_v3 python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > $O/ncu_f.log 2>&1
python tools/ncu_summ.py $O/fused_v3.ncu-rep > $O/ncu_fused_v3.txt 2>&1
python tools/sass_blocks.py $O/fused_v3.ncu-rep deposit_current_kernel_v3 >> $O/ncu_fused_v3.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_v3 -s 3 -c 1 -o $O/fused_cic python bench.py --steps 3 --order 1 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > $O/ncu_c.log 2>&1
python tools/ncu_summ.py $O/fused_cic.ncu-rep > $O/ncu_fused_cic.txt 2>&1
python tools/sass_blocks.py $O/fused_cic.ncu-rep deposit_current_kernel_v3 >> $O/ncu_fused_cic.txt 2>&1
timeout 600 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c3o3 --no-cpu-baseline --steps 5 > $O/bench_c3o3.json 2> $O/bench_c3o3.err
timeout 600 python bench.py --slab --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_slab.json 2> $O/bench_slab.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() { ncu --metrics $M --clock-control none -k regex:deposit_current_kernel -c 12 --csv --log-file gpurun_out/traffic/$1.csv python bench.py $2 --steps 4 --warmup 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/traffic/$1.log 2>&1; }
run c2_o3 "--config c2"
run c2_o2 "--config c2 --order 2"
run c2_o1 "--config c2 --order 1"
run c1_o1 "--config c1"
run c4_o3 "--config c4"
