#!/bin/bash
# Drop-in proof: the reference's own pkg/tests against the patched package.
# In the build container first run:  scripts/run_reference_suite.sh --stage
# (copies /root/reference/pkg into baseline/_ref/pkg, git-ignored, travels with gpurun)
set -e
cd "$(dirname "$0")/.."
if [ "$1" = "--stage" ]; then
  rm -rf baseline/_ref/pkg && mkdir -p baseline/_ref && cp -r /root/reference/pkg baseline/_ref/pkg
  echo staged; exit 0
fi
[ -d baseline/_ref/pkg ] || { echo "baseline/_ref/pkg missing (stage it first)"; exit 0; }
mkdir -p gpurun_out
WORK=$(mktemp -d)
cp -r baseline/_ref/pkg "$WORK/pkg"
ROOTDIR=$(pwd)
cd "$WORK/pkg"
PYTHONPATH="$ROOTDIR:$ROOTDIR/scripts/refsuite:$WORK/pkg/src:$WORK/pkg/tests" \
  timeout 3000 python -m pytest tests -p vmp_patch_plugin -p no:cacheprovider -q -rf --durations=15 ${REF_ARGS:-} \
  > "$ROOTDIR/gpurun_out/reference_suite.log" 2>&1
echo "reference suite rc=$?" >> "$ROOTDIR/gpurun_out/reference_suite.log"
tail -5 "$ROOTDIR/gpurun_out/reference_suite.log"
