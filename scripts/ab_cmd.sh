# A/B of the config-2 step: a previous tree copied to ab_old/ (git-ignored) vs this one
mkdir -p gpurun_out
for pass in 1 2; do
 for d in ab_old .; do
  echo "== $d pass $pass" >> gpurun_out/ab.log
  (cd $d && timeout 300 python scripts/exp_flush.py 2>&1 | tail -2) >> gpurun_out/ab.log
 done
done
cat gpurun_out/ab.log
