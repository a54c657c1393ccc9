mkdir -p gpurun_out
for o in 3 1; do python tools/jbench.py $o 128 16; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rho.csv -k regex:"density|fill_holes" python tools/jbench.py 3 128 16 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"density_rows" -s 2 -c 1 -o gpurun_out/full_rho python tools/jbench.py 3 128 16 > /dev/null 2>&1
