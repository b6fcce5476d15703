#!/bin/bash
mkdir -p gpurun_out
python scripts/profile_kernels.py cfg1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"vmp_validate" -s 1 -c 1 -o gpurun_out/prof_cfg1 python scripts/profile_kernels.py cfg1 > gpurun_out/ncu_cfg1.log 2>&1
tail -2 gpurun_out/ncu_cfg1.log
