#!/bin/bash
# ncu evidence for one round (run under gpurun, 1 GPU). Output: gpurun_out/<tag>_*.
tag=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${tag}_launches_bench.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FwdTraits -s 30 -c 1 -o gpurun_out/${tag}_fwd $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:BwdTraits -s 30 -c 1 -o gpurun_out/${tag}_bwd $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:CeTraits -s 0 -c 2 -o gpurun_out/${tag}_ce $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:GenTraits -s 12 -c 2 -o gpurun_out/${tag}_gen $B > /dev/null 2>&1
ls -la gpurun_out | grep $tag
