# rho v2 (thread = (X, jy), z-chains, staged sy*sz): parity + timing vs v1
set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "not test_c3_geometry and not test_c2_full" 2>&1 | tail -8 > gpurun_out/rho_pytest.log
for o in 3 2 1; do timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/rho_jbench.log 2>&1; PICGPU_RHO_V1=1 timeout 120 python tools/jbench.py $o 128 16 >> gpurun_out/rho_jbench.log 2>&1; done
python tools/jbench.py 3 128 16 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:density_blocks2 -s 1 -c 1 -o gpurun_out/rho2 python tools/jbench.py 3 128 16 > gpurun_out/rho_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x 2>&1 | tail -5 > gpurun_out/rho_cfg.log
