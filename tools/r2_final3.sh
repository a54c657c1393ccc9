# Final-tree validation and profiles (r02, second half): GPU suite, smoke, default bench (timed), reference arm,
# launch list of the bench command, ncu --set full of the fused kernel and of the mover kernels, other configs.
set -x
O=gpurun_out/f3
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
( time timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -8 ) > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time timeout 900 python bench.py ) > $O/bench_c2.json 2> $O/bench_c2.err
( time timeout 900 python bench.py --impl reference ) > $O/bench_ref.json 2> $O/bench_ref.err
bash tools/ab_lib.sh paper_2601_08277_b200/libpicgpu.so build/libpicgpu_ppb2.so > $O/ppb2_ab.txt 2>&1
python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 20 --warmup 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > $O/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:deposit_current_kernel_v3 -s 3 -c 1 -o $O/fused_v3 python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > $O/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_movers|k_insert" -s 6 -c 2 -o $O/movers python bench.py --steps 3 --no-orders --no-cpu-baseline --e2e-steps 0 --steady-steps 0 > $O/ncu_m.log 2>&1
python tools/ncu_summ.py $O/fused_v3.ncu-rep > $O/ncu_fused_v3.txt 2>&1
python tools/sass_blocks.py $O/fused_v3.ncu-rep deposit_current_kernel_v3 >> $O/ncu_fused_v3.txt 2>&1
python tools/ncu_summ.py $O/movers.ncu-rep > $O/ncu_movers.txt 2>&1
python tools/sass_blocks.py $O/movers.ncu-rep k_movers 400000 >> $O/ncu_movers.txt 2>&1
timeout 600 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c3o3 --no-cpu-baseline --steps 5 > $O/bench_c3o3.json 2> $O/bench_c3o3.err
timeout 600 python bench.py --slab --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_slab.json 2> $O/bench_slab.err
bash tools/traffic.sh > $O/traffic.log 2>&1
python tools/traffic_json.py > $O/traffic.json 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
