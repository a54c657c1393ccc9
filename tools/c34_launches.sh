# per-kernel launch lists of the C3 sort profile and a short C4 bench, for the lib in $PICGPU_LIB (default in-tree)
tag=${1:-cur}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_$tag.csv python tools/c3_sort_prof.py > gpurun_out/c3_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_$tag.csv python bench.py --config c4 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/c4_$tag.log 2>&1
tail -2 gpurun_out/c3_$tag.log
