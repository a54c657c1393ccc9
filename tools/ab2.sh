bash tools/ab_env.sh PICGPU_INSERT_BLOCKS 4 16
bash tools/ab_env.sh PICGPU_MOVERS_BLOCKS 4 16
