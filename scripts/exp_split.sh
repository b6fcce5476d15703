# config-1 kernel variants: split 1 / 2, streamed (graph per batch / one graph) vs single flushed launches
mkdir -p gpurun_out
for s in 1 2; do echo "== split $s" >> gpurun_out/split.log; VMP_EXP_SPLIT=$s timeout 300 python scripts/exp_stream.py cfg1 >> gpurun_out/split.log 2>&1; done
timeout 300 python scripts/exp_stream.py cfg3 cfg4 >> gpurun_out/split.log 2>&1
cat gpurun_out/split.log
