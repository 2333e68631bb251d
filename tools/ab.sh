#!/bin/bash
# A/B of env toggles on the same box: tools/ab.sh "ENV=1" "" ... (each arg: env assignments for one bench run)
for cfg in "$@"; do
  v=$(env $cfg python bench.py --no-cpu-baseline --steps 20 --warmup 10 --e2e-steps 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['kernel_ms_per_step']
e=d.get('energy',{})
print(round(d['value']), round(d['ms_per_step'],3), 'sm', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), 'J/step', round(e.get('j_per_step',0),2), 'W', round(e.get('power_w_avg',0)),
      {x: round(k[x],3) for x in ('gemm_rec_fwd','gemm_rec_bwd','gemm_wgrad','gemm_dgrad_x','gemm_out') if x in k})")
  echo "[$cfg] $v"
done
