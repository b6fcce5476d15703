#!/bin/bash
# Motion parity tests on the current tree, then the A/B of the config-2 step
# against ab_old/ (scripts/ab_cmd.sh).   VARIANTS as in ab_cmd.sh.
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_graphs.py -q -x -m gpu -k "${TESTS:-rake or motion or cfg2 or workspace or edge}" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
tail -3 gpurun_out/pytest_ab.log
bash scripts/ab_cmd.sh
