#!/bin/bash
# Instruction-counter capture of the culled FP32 path's kernels (fused_trace,
# fused_sample) for one configuration: FP32/FP64 thread instructions by
# opcode (paired FFMA2/FADD2/FMUL2 counted separately), pipe activity,
# occupancy, divergence, DRAM bytes.  Feeds tools/ncu_flops.py ->
# profiles/ncu_flops.json (bench.py roofline.counter_*).
#   tools/ncu_counters.sh C2 gpurun_out/ctr_C2.csv
set -e
CFG=${1:-C2}
OUT=${2:-gpurun_out/ctr_$CFG.csv}
M=gpu__time_duration.sum
for op in ffma ffma2 fadd fadd2 fmul fmul2 dfma dadd dmul; do
  M=$M,sm__sass_thread_inst_executed_op_${op}_pred_on.sum
done
M=$M,sm__inst_executed.sum,smsp__thread_inst_executed.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum
M=$M,sm__inst_executed_pipe_fp64.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size,launch__occupancy_limit_registers
python tools/profile_frame.py --config "$CFG" --frames 4 > /dev/null
ncu --metrics "$M" --clock-control none -k regex:fused_ -s 2 -c 4 --csv --log-file "$OUT" \
    python tools/profile_frame.py --config "$CFG" --frames 4 > /dev/null
