#!/bin/bash
# motion parity, then A/B of codegen switches on the config-2 step (back-to-back + flushed), then the timeline
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_graphs.py tests/test_gpu_cabi.py -q -x -m gpu -k "rake or motion or cfg2 or workspace or edge or cabi" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
tail -4 gpurun_out/pytest_ab.log
for pass in 1 2; do
  for c in "$@"; do
    echo "== $c" >> gpurun_out/ab.log
    env $c timeout 300 python scripts/exp_flush.py 2>&1 | grep -E "^flush|back-to-back" | tail -3 >> gpurun_out/ab.log
  done
done
cat gpurun_out/ab.log
bash scripts/trace_ab.sh > /dev/null
