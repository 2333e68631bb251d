#!/bin/bash
# Full ncu capture of one kernel instance inside a 1-step bench run (1 GPU).
# Usage: tools/ncu_one.sh <tag> <kernel-regex> <skip-count>
tag=$1; re=$2; skip=${3:-0}
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -s $skip -c 1 \
    -o gpurun_out/${tag} python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${tag}.log 2>&1
ls -la gpurun_out/${tag}.ncu-rep
