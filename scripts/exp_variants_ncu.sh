#!/bin/bash
# ncu --set full of one workload per codegen variant (VMP_EXP), raw CSV + source page kept.
#   VARIANTS="nopack,coarse -" WHAT="cfg3" bash scripts/exp_variants_ncu.sh
mkdir -p gpurun_out
for v in $VARIANTS; do
  e=$v; [ "$v" = "-" ] && e=""; tag=${v//,/_}; [ "$v" = "-" ] && tag=default
  for w in $WHAT; do
    re="vmp_validate"; [ "$w" = "motion" ] && re="vmp_motion_p"
    VMP_EXP=$e python scripts/profile_kernels.py $w > /dev/null 2>&1 && \
    VMP_EXP=$e ncu --set full --clock-control none --import-source on -k regex:"$re" -s 1 -c 1 \
        -o gpurun_out/var_${w}_$tag -f python scripts/profile_kernels.py $w > gpurun_out/ncu_var.log 2>&1
    ncu -i gpurun_out/var_${w}_$tag.ncu-rep --page raw --csv > gpurun_out/var_${w}_$tag.raw.csv 2>/dev/null
    ncu -i gpurun_out/var_${w}_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/var_${w}_$tag.src.csv 2>/dev/null
    rm -f gpurun_out/var_${w}_$tag.ncu-rep
  done
done
ls -la gpurun_out | tail
