#!/bin/bash
# ncu evidence for one round (run under gpurun, 1 GPU). Output: gpurun_out/<tag>_*.
tag=${1:-r01}
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${tag}_launches_bench.log 2>&1
# one full capture of a large tcgen05 GEMM launch (wgrad-shaped) and of the recurrent-step GEMM
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 40 -c 3 \
    -o gpurun_out/${tag}_gemm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/${tag}_gemm_bench.log 2>&1
ls -la gpurun_out
