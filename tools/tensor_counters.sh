#!/bin/bash
# Tensor-pipe counters of every kernel in one bench step (1 GPU, under gpurun). Output:
# gpurun_out/<tag>_tensor.csv; summarise with tools/tensor_counters.py.
#   sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32   math ops issued by UTCHMMA (bf16 -> fp32)
#   ... .sum.pct_of_peak_sustained_elapsed            the same as a share of the tensor pipe's peak
#   sm__pipe_tensor_cycles_active_realtime             the counter DESIGN §6 found unstable
#   sm__inst_executed_pipe_tensor_subpipe_hmma         UTCHMMA warp instructions
tag=${1:-r02c}
M=gpu__time_duration.sum,launch__grid_size
M=$M,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum
M=$M,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed
M=$M,sm__inst_executed_pipe_tensor_subpipe_hmma.sum
M=$M,sm__cycles_elapsed.avg.per_second
ncu --metrics $M --clock-control none -c 700 --csv --log-file gpurun_out/${tag}_tensor.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${tag}_tensor_bench.log 2>&1
