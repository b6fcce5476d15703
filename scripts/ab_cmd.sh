# A/B: e2e of the current bench.py vs the round-1 bench protocol (scripts/bench_old_exp.py) on this tree
mkdir -p gpurun_out
for pass in 1 2 3; do
  for b in bench.py scripts/bench_old_exp.py; do
    echo "== $b pass $pass" >> gpurun_out/ab.log
    timeout 300 python $b --steps 20 --warmup 5 --no-aux --no-cpu-baseline 2>&1 \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], round(d['value']/1e6, 2), round(d['e2e']['value']/1e6, 2))" >> gpurun_out/ab.log
  done
done
timeout 300 python scripts/exp_flush.py 2>&1 | tail -1 >> gpurun_out/ab.log
cat gpurun_out/ab.log
