mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"density_blocks" -s 2 -c 1 -o gpurun_out/full_rho python tools/jbench.py 3 128 16 > /dev/null 2>&1
