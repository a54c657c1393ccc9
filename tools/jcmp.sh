# J kernel A/B: v3 (default) vs v1 at C2, orders 3 and 2
for o in 3 2; do
  python tools/jbench.py $o 128 16 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v3', d['order'], round(d['deposit_current_ms'],4))"
  PICGPU_J_LANE=v1 python tools/jbench.py $o 128 16 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v1', d['order'], round(d['deposit_current_ms'],4))"
done
