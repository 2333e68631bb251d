#!/bin/bash
# A/B of env toggles at a given model width: tools/ab_shape.sh <hidden> "ENV=1" "" ...
h=$1; shift
for cfg in "$@"; do
  v=$(env $cfg python bench.py --hidden $h --no-cpu-baseline --steps 20 --warmup 10 --e2e-steps 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['kernel_ms_per_step']
print(round(d['value']), round(d['ms_per_step'],3), 'sm', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'),
      {x: round(k[x],3) for x in ('gemm_rec_fwd','gemm_rec_bwd','gemm_wgrad','gemm_dgrad_x','gemm_out') if x in k})")
  echo "[H=$h $cfg] $v"
done
