#!/bin/bash
# Full ncu captures of selected kernels (1 GPU). Usage: tools/ncu_kernels.sh <tag>
tag=${1:-k}
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:BwdTraits -s 5 -c 1 -o gpurun_out/${tag}_bwd $B > gpurun_out/${tag}_bwd.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FwdTraits -s 30 -c 1 -o gpurun_out/${tag}_fwd $B > gpurun_out/${tag}_fwd.log 2>&1
# (output GEMM captured separately)
ls -la gpurun_out
