#!/bin/bash
# A/B of the rake's environment-copy overlap (VMP_EXP=waitenv = wait up front), motion parity, timeline
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_graphs.py -q -x -m gpu -k "rake or motion or cfg2 or workspace or edge" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
tail -3 gpurun_out/pytest_ab.log
bash scripts/exp_ab.sh "VMP_EXP=waitenv" "X=1"
bash scripts/trace_ab.sh
