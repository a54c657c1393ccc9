set -x
mkdir -p gpurun_out/rho3
timeout 900 python -m pytest tests -q -m gpu -x -k "density or rho or golden or c1_full or lwfa" 2>&1 | tail -5 > gpurun_out/rho3/pytest.log
for o in 3 2 1; do timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/rho3/jbench.log 2>&1; PICGPU_LIB=build/libpicgpu_rs0.so timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/rho3/jbench.log 2>&1; done
python tools/jbench.py 3 128 16 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:density_blocks -s 1 -c 1 -o gpurun_out/rho3/rho_syz python tools/jbench.py 3 128 16 > gpurun_out/rho3/ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "c2_full" 2>&1 | tail -3 > gpurun_out/rho3/cfg.log
