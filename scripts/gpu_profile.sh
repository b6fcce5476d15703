#!/bin/bash
# ncu evidence: launch list of the bench + full captures of the top kernels.
# Each capture runs only after the same command exited 0 without ncu.
#   bash scripts/gpu_profile.sh [names...]   (default: all)
mkdir -p gpurun_out
want() { [ $# -eq 0 ] || [[ " $WANT " == *" $1 "* ]]; }
WANT="$*"
if [ -z "$WANT" ] || [[ " $WANT " == *" launches "* ]]; then
  B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
  $B > gpurun_out/plain_bench.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
        --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
fi
cap() {  # cap <name> <kernel regex> <profile_kernels args...>
  local name=$1 re=$2; shift 2
  if [ -n "$WANT" ] && [[ " $WANT " != *" $name "* ]]; then return; fi
  python scripts/profile_kernels.py "$@" > gpurun_out/plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$re" -s 1 -c 1 \
      -o gpurun_out/prof_$name python scripts/profile_kernels.py "$@" > gpurun_out/ncu_$name.log 2>&1
  # raw metrics as CSV (small) and the executed FP32 flop (SASS source page)
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/raw_$name.csv 2>/dev/null
  python scripts/executed_flops.py gpurun_out/prof_$name.ncu-rep > gpurun_out/exec_$name.json 2>/dev/null
}
cap motion "vmp_motion_p" motion
cap begin "motion_begin" motion
cap finalize "motion_finalize" motion
cap cfg1 "vmp_validate" cfg1
cap cfg3 "vmp_validate" cfg3
cap cfg3_dense "vmp_validate" cfg3 --dense
cap cfg4 "vmp_validate" cfg4
cap cfg4_dense "vmp_validate" cfg4 --dense
cap cfg5_1024 "vmp_validate" cfg5_1024
cap fk "vmp_fk_spheres" fk
cap knn "vmp_k_knn" knn
python scripts/ncu_summary.py gpurun_out/prof_*.ncu-rep > gpurun_out/ncu_summary.md 2>/dev/null
# the .ncu-rep files themselves only where KEEP lists them (gpurun brings back at most 64 MiB)
for f in gpurun_out/prof_*.ncu-rep; do
  name=${f#gpurun_out/prof_}; name=${name%.ncu-rep}
  if [[ " ${KEEP:-motion cfg1 cfg3} " != *" $name "* ]]; then rm -f $f; fi
done
ls -la gpurun_out/
