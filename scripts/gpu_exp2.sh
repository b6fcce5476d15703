#!/bin/bash
# dynamic-queue rake vs planned rake: motion parity, A/B (guard variants), timeline
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_graphs.py tests/test_gpu_cabi.py -q -x -m gpu -k "rake or motion or cfg2 or workspace or edge or cabi" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
tail -15 gpurun_out/pytest_ab.log
bash scripts/exp_ab.sh "VMP_MOTION_PLAN=1" "X=1" "VMP_EXP_GUARD=2" "VMP_EXP_GUARD=1" "VMP_EXP_GUARD=0"
bash scripts/trace_ab.sh
