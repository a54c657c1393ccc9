# iteration check on one B200: GPU tests, J-only per order, the C2 bench, ncu of the pencil kernels
set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/it_pytest.log
for o in 3 2 1; do timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/it_jbench.log 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
if [ "$1" = "ncu" ]; then
python tools/jbench.py 3 128 16 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_pencil -s 4 -c 1 -o gpurun_out/it_j python tools/jbench.py 3 128 16 > gpurun_out/it_ncu.log 2>&1
python bench.py --steps 3 --warmup 3 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_pencil -s 3 -c 1 -o gpurun_out/it_fused python bench.py --steps 3 --warmup 3 > gpurun_out/it_ncu2.log 2>&1
fi
