timeout 900 python -m pytest tests -m gpu -x -q -k "density or rho or lockstep or fused or golden or slab" 2>&1 | tail -3
for o in 3 2 1; do python tools/jbench.py $o 128 16; done
for o in 3 1; do PICGPU_RHO_ROWS=1 python tools/jbench.py $o 128 16; done
