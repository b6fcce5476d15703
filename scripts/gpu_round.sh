#!/bin/bash
# One gpurun call of round-end evidence: GPU tests, smoke, the bench (ours + the
# reference arm), the config-5 sweep and the reference's own suite patched onto
# the B200 path.  Outputs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 1200 python scripts/sweep_cfg5.py > gpurun_out/sweep_cfg5.jsonl 2> gpurun_out/sweep_cfg5.err; echo "sweep rc=$?" >> gpurun_out/sweep_cfg5.err
bash scripts/run_reference_suite.sh > /dev/null 2>&1
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/reference_suite.log gpurun_out/sweep_cfg5.err
