# J kernel A/B: v3 (default) vs v1; args: "order n ppc" triples
for cfg in "$@"; do
  set -- $cfg
  a=$(python tools/jbench.py $1 $2 $3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['deposit_current_ms'],4))")
  b=$(PICGPU_J_LANE=v1 python tools/jbench.py $1 $2 $3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['deposit_current_ms'],4))")
  echo "order $1 n $2 ppc $3: v3 $a ms  v1 $b ms"
done
