#!/bin/bash
# A/B of env toggles on the same box: tools/ab.sh "ENV=1" "" ... (each arg: env assignments for one bench run)
for cfg in "$@"; do
  v=$(env $cfg python bench.py --no-cpu-baseline --steps 20 --warmup 10 --e2e-steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})")
  echo "[$cfg] $v"
done
