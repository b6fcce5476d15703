mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mp.csv python scripts/profile_kernels.py motion > gpurun_out/mp.log 2>&1
grep gpu__time_duration gpurun_out/mp.csv | awk -F'","' '{print $5, $NF}' | head -12
