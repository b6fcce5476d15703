#!/bin/bash
mkdir -p gpurun_out
python scripts/profile_kernels.py motion > gpurun_out/plain_motion.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/motion_launches.csv python scripts/profile_kernels.py motion > gpurun_out/ncu_ml.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"vmp_motion_p" -s 1 -c 1 -o gpurun_out/prof_motion2 python scripts/profile_kernels.py motion > gpurun_out/ncu_m2.log 2>&1
cat gpurun_out/motion_launches.csv | tail -40
