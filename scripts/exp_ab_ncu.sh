#!/bin/bash
# ncu --set full of the config-2 rake under two codegen experiment settings
# usage: bash scripts/exp_ab_ncu.sh "<envA>" "<envB>"
mkdir -p gpurun_out
i=0
for c in "$1" "$2"; do
  env $c python scripts/profile_kernels.py motion > /dev/null 2>&1 && \
  env $c ncu --set full --clock-control none --import-source on -k regex:"vmp_motion_p" -s 1 -c 1 \
      -o gpurun_out/ab_$i python scripts/profile_kernels.py motion > gpurun_out/ab_ncu_$i.log 2>&1
  i=$((i+1))
done
ls gpurun_out
