#!/bin/bash
# A/B of environment switches on the bench: step, e2e, fkcc ms, parity.  usage: gpu_ab_bench.sh "<env1>" "<env2>" ...
mkdir -p gpurun_out
rm -f gpurun_out/ab3.log
for pass in 1 2; do
for e in "$@"; do
  echo "== $e" >> gpurun_out/ab3.log
  env $e timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
f=d['fkcc']
print('step', d['ms_per_step'], 'e2e', round(d['e2e']['value']/1e6,1), ' '.join(f'{k}:{f[k][\"product\"][\"ms\"]}/{f[k][\"streamed\"][\"ms\"]}' for k in ('cfg1','cfg3','cfg4')), 'parity', [d['parity'][k].get('mismatches_outside_band', d['parity'][k].get('mismatches')) for k in d['parity']])
" >> gpurun_out/ab3.log
done
done
cat gpurun_out/ab3.log
