for v in c0u1m6 c1u1m8 c0u1m4 c1u1m6 c0u2m4; do echo "== $v"; PICGPU_LIB=build/libpicgpu_$v.so python tools/step_timing.py 2>&1 | tail -1; done
PICGPU_LIB=build/libpicgpu_c0u1m6.so timeout 300 ncu --set full --clock-control none -k regex:"k_push" -c 1 -o gpurun_out/push_p2 python tools/step_timing.py > /dev/null 2>&1
