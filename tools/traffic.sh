# DRAM bytes per launch of the dominant J kernel for every bench config/order/path
# (ncu, --clock-control none) -> gpurun_out/traffic/*.csv; tools/traffic_json.py -> profiles/ncu_traffic.json
mkdir -p gpurun_out/traffic
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() {  # name, bench args
  ncu --metrics $M --clock-control none -k regex:deposit_current_kernel -c 12 --csv --log-file gpurun_out/traffic/$1.csv \
      python bench.py $2 --steps 4 --warmup 3 --no-orders --no-cpu-baseline --e2e-steps 0 > gpurun_out/traffic/$1.log 2>&1
}
run c2_o3 "--config c2"
run c2_o2 "--config c2 --order 2"
run c2_o1 "--config c2 --order 1"
run c1_o1 "--config c1"
run c4_o3 "--config c4"
run c3o3_o3 "--config c3o3"
run c3o1_o1 "--config c3o1"
run c3o2_o2 "--config c3o2"
