#!/bin/bash
# A/B of c5 variants inside one GPU call: bash scripts/c5_ab.sh rounds "name:ENV=VAL,ENV2=VAL2 ..." -> batch-it/s per variant
rounds=${1:-2}; shift
for i in $(seq $rounds); do
  for spec in "$@"; do
    name=${spec%%:*}; envs=${spec#*:}
    ( IFS=','; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done
      python bench.py --workload c5 --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$name', round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1))" )
  done
done
