#!/bin/bash
# A/B timing of the config-2 step: 200 back-to-back replays (scripts/exp_flush.py)
# per variant, each variant an env assignment list (e.g. VMP_MOTION_CAPPED=0),
# two interleaved passes.   usage: bash scripts/exp_ab.sh "<env1>" "<env2>" ...
mkdir -p gpurun_out
for pass in 1 2; do
  for c in "$@"; do
    echo "== $c" >> gpurun_out/ab.log
    env $c timeout 300 python scripts/exp_flush.py 2>&1 | grep back-to-back | tail -2 >> gpurun_out/ab.log
  done
done
cat gpurun_out/ab.log
