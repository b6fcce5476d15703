# per-item rake timeline of this tree (and of ab_old/ when given "old")
mkdir -p gpurun_out
VMP_MOTION_TRACE=1 timeout 300 python scripts/exp_motion_trace.py > gpurun_out/trace_new.log 2>&1
cp gpurun_out/motion_items.npz gpurun_out/motion_items_new.npz
if [ "$1" = old ]; then
(cd ab_old && mkdir -p gpurun_out && VMP_MOTION_TRACE=1 timeout 300 python scripts/exp_motion_trace.py > ../gpurun_out/trace_old.log 2>&1; cp gpurun_out/motion_items.npz ../gpurun_out/motion_items_old.npz)
fi
cat gpurun_out/trace_new.log
