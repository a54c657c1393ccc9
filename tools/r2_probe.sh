set -x
mkdir -p gpurun_out/probe
PICGPU_FUSE_MAX_MOVED=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --clock-control none -k regex:"k_movers|k_insert|k_borrow|deposit_current_kernel|k_departures|k_push" --csv --log-file gpurun_out/probe/c3_fused_launches.csv python bench.py --config c3o3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/probe/c3ncu.log 2>&1
