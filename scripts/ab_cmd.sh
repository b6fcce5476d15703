# A/B of the config-2 step: directories / environment variants, e.g.
#   VARIANTS="ab_old:X=1 .:X=1 .:VMP_NO_FFMA2=1" bash scripts/ab_cmd.sh
# ab_old/ = a previous tree (git-ignored).  Per variant and pass: 200 back-to-back
# steps (scripts/exp_flush.py) and the flushed steps / e2e of the round-1 bench
# protocol (scripts/bench_old_exp.py in this tree, bench.py in ab_old/).
mkdir -p gpurun_out
VARIANTS=${VARIANTS:-"ab_old:X=1 .:X=1"}
for pass in 1 2; do
  for v in $VARIANTS; do
    d=${v%%:*}; e=${v#*:}
    b=bench.py; [ "$d" = "." ] && b=scripts/bench_old_exp.py
    echo "== $v pass $pass" >> gpurun_out/ab.log
    (cd $d && env $(echo $e | tr , ' ') timeout 300 python scripts/exp_flush.py 2>&1 | tail -1) >> gpurun_out/ab.log
    (cd $d && env $(echo $e | tr , ' ') timeout 300 python $b --steps 20 --warmup 5 --no-aux --no-cpu-baseline 2>&1 \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], round(d['value']/1e6, 2), round(d['e2e']['value']/1e6, 2))") >> gpurun_out/ab.log
  done
done
cat gpurun_out/ab.log
