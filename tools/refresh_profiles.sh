#!/bin/bash
# Round evidence (1 GPU, under gpurun): launch list of one step, full ncu captures of the top
# kernels, and a bench line. Output: gpurun_out/<tag>_*. Summarise locally with
#   python tools/summarize_ncu.py <tag> gpurun_out/<tag>_*.ncu-rep --launches gpurun_out/<tag>_launches.csv
tag=${1:-r02}
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 700 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/${tag}_launches_bench.log 2>&1
cap() {  # name regex skip count
  ncu --set full --metrics sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum.pct_of_peak_sustained_elapsed \
      --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c ${4:-1} \
      -o gpurun_out/${tag}_$1 $B > gpurun_out/${tag}_$1.log 2>&1
}
cap fwd "FwdPersistT" 2
cap bwd "BwdPersistTraits" 2
cap ce "CeTraits" 0 2
cap wgrad "GenTraits<.int.256, .bool.1, .bool.1, .bool.0, .int.0, .bool.0, .bool.0>" 2
cap wsplit "GenTraits<.int.256, .bool.1, .bool.1, .bool.0, .int.2, .bool.1" 0
cap dgrad "GenTraits<.int.512" 0
cap update "sdpsgd_kernel" 0
cap gather "gather_kernel" 1
python bench.py > gpurun_out/${tag}_bench.log 2>&1
python tools/ingress_probe.py > gpurun_out/${tag}_ingress.txt 2>&1  # (its A operand is DRAM-streamed: see DESIGN 6)
[ -x tools/tma_mc_probe ] && timeout 120 tools/tma_mc_probe 32 40 > gpurun_out/${tag}_tma_probe.txt 2>&1
[ -x tools/mma_rate ] && timeout 120 tools/mma_rate > gpurun_out/${tag}_mma_rate.txt 2>&1
tail -1 gpurun_out/${tag}_bench.log > gpurun_out/${tag}_bench.json
ls -la gpurun_out | grep $tag
