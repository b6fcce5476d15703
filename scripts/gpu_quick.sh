#!/bin/bash
# quick loop: motion parity tests + bench (no aux) + launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rake or cfg2 or motion or discretize" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-aux --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
python scripts/profile_kernels.py motion > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/motion_launches.csv python scripts/profile_kernels.py motion > /dev/null 2>&1
tail -2 gpurun_out/pytest_quick.log; tail -c 600 gpurun_out/bench_quick.log
