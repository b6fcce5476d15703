#!/bin/bash
# ncu counters for the config-5 sweep points at N = 2^20 (and configs 3 / 4):
# executed FP32 instructions (-> executed GFLOP/s), FMA-pipe utilisation,
# issue activity and DRAM bytes, product and dense mode.
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for w in cfg5_16 cfg5_128 cfg5_1024 cfg3 cfg4; do
  for d in "" "--dense"; do
    tag=$w${d:+_dense}
    python scripts/profile_kernels.py $w $d --reps 2 > gpurun_out/plain_$tag.log 2>&1 && \
    ncu --metrics $M --clock-control none -k regex:"vmp_validate" -s 1 -c 1 --csv \
        python scripts/profile_kernels.py $w $d --reps 2 > gpurun_out/sweep_ncu_$tag.csv 2>&1
  done
done
ls gpurun_out/sweep_ncu_*
