for v in b64 b16 b32 b128; do
  echo "== $v"; PICGPU_LIB=build/libpicgpu_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bpb_$v.csv -k regex:"relayout|fill_slack" python tools/shift_timing.py 0.06 > /dev/null 2>&1
  python tools/launches.py gpurun_out/bpb_$v.csv
done
