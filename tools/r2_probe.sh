set -x
mkdir -p gpurun_out/probe
bash tools/ab_cfgs.sh paper_2601_08277_b200/libpicgpu.so build/libpicgpu_stcs.so > gpurun_out/probe/stcs.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/probe/pytest.log
