#!/bin/bash
# A/B of codegen switches (VMP_EXP) on the bench: step, e2e, fkcc ms.  usage: gpu_exp3.sh "<exp1>" "<exp2>" ...
mkdir -p gpurun_out
rm -f gpurun_out/ab3.log
for pass in 1 2; do
for e in "$@"; do
  echo "== VMP_EXP=$e" >> gpurun_out/ab3.log
  VMP_EXP=$e timeout 300 python scripts/exp_flush.py 2>&1 | grep back-to-back | tail -1 >> gpurun_out/ab3.log
  VMP_EXP=$e timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
f=d['fkcc']
print('step', d['ms_per_step'], 'e2e', round(d['e2e']['value']/1e6,1), ' '.join(f'{k}:{f[k][\"product\"][\"ms\"]}/{f[k][\"streamed\"][\"ms\"]}' for k in ('cfg1','cfg3','cfg4')), 'parity', [d['parity'][k].get('mismatches_outside_band', d['parity'][k].get('mismatches')) for k in d['parity']])
" >> gpurun_out/ab3.log
done
done
cat gpurun_out/ab3.log
