#!/bin/bash
# A/B of codegen experiment variants (VMP_EXP) on one box: bench.py per variant,
# two interleaved passes.  usage: VARIANTS="nopack,coarse nopack - coarse" bash scripts/exp_variants_run.sh
mkdir -p gpurun_out; rm -f gpurun_out/variants.log
for pass in 1 2; do
  for v in $VARIANTS; do
    e=$v; [ "$v" = "-" ] && e=""
    VMP_EXP=$e timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2> gpurun_out/variants.err | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
f = d['fkcc']
print('$v pass $pass: rake ms %.4f e2e %.1fM |' % (d['ms_per_step'], d['e2e']['value'] / 1e6),
      ' | '.join('%s prod %.4f dense %.4f strm %.4f' % (c, f[c]['product']['ms'], f[c]['dense']['ms'], f[c]['streamed']['ms']) for c in ('cfg1', 'cfg3', 'cfg4')),
      '| mism', [d['parity'][c].get('mismatches_outside_band', d['parity'][c].get('mismatches')) for c in ('cfg1', 'cfg2', 'cfg3', 'cfg4')])
" >> gpurun_out/variants.log
  done
done
cat gpurun_out/variants.log
