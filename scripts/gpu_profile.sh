#!/bin/bash
# ncu evidence: launch list of the bench + full captures of the top kernels.
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
for w in motion cfg3 cfg4; do
  python scripts/profile_kernels.py $w > gpurun_out/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"vmp_(motion|validate)" -s 1 -c 1 \
      -o gpurun_out/prof_$w python scripts/profile_kernels.py $w > gpurun_out/ncu_$w.log 2>&1
done
python scripts/profile_kernels.py cfg3 --dense > gpurun_out/plain_cfg3d.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"vmp_validate" -s 1 -c 1 \
      -o gpurun_out/prof_cfg3_dense python scripts/profile_kernels.py cfg3 --dense > gpurun_out/ncu_cfg3d.log 2>&1
python scripts/profile_kernels.py fk > gpurun_out/plain_fk.log 2>&1 && \
  ncu --set full --clock-control none -k regex:"vmp_fk" -s 1 -c 1 \
      -o gpurun_out/prof_fk python scripts/profile_kernels.py fk > gpurun_out/ncu_fk.log 2>&1
ls -la gpurun_out/
