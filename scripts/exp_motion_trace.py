"""Timeline of one config-2 rake launch (run with VMP_MOTION_TRACE=1): when CTAs
start, when the plan is ready, when each warp finds the queue empty, CTA exit,
and per-item records (a debug build of the rake: VMP_MOTION_TRACE_ITEMS=1 is
set here before codegen runs, so the module is compiled by NVRTC on first use).

    VMP_MOTION_TRACE=1 python scripts/exp_motion_trace.py
"""
import ctypes
import os
import sys
from pathlib import Path

os.environ["VMP_MOTION_TRACE_ITEMS"] = "1"

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, workloads  # noqa: E402
from paper_2309_14545_b200 import motion as M  # noqa: E402
from paper_2309_14545_b200._native import lib  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
mw = workloads.config2()
rob = load_robot(mw.robot)
ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
mv = M.MotionValidator(ctx, len(mw.starts), mw.resolution, width=32)
mv(mw.starts, mw.goals)
for _ in range(3):
    mv()
torch.cuda.synchronize()
flush.zero_()
torch.cuda.synchronize()
mv()
torch.cuda.synchronize()
buf = np.zeros(1 << 16, dtype=np.uint64)
n = lib().vmp_debug_motion_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
tr = buf[:min(n, 8192)].reshape(-1, 8).astype(np.int64)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
rel = (tr[:, :7] - t0) / 1e3
print(f"CTAs traced: {len(tr)}, items taken: {int(tr[:, 7].sum())}")
for name, col in (("entry", 0), ("plan ready", 1), ("exit", 6)):
    c = rel[:, col]
    print(f"{name:12s}: min {c.min():7.2f}  median {np.median(c):7.2f}  p90 {np.percentile(c, 90):7.2f}  max {c.max():7.2f} us")
w = rel[:, 2:6].ravel()
print(f"{'warp done':12s}: min {w.min():7.2f}  p10 {np.percentile(w, 10):7.2f}  median {np.median(w):7.2f}  p90 {np.percentile(w, 90):7.2f}  max {w.max():7.2f} us")
hist, edges = np.histogram(w, bins=12)
print("warp-done histogram:", ", ".join(f"{e:.0f}us:{h}" for e, h in zip(edges, hist)))
items = tr[:, 7]
print(f"items per CTA: min {items.min()} median {np.median(items):.0f} max {items.max()}")

# per-item records (start, end, round << 32 | edge, warp << 48 | loop top) of the last launch
buf = np.zeros(1 << 17, dtype=np.uint64)
n = lib().vmp_debug_motion_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
rec = buf[8192:8192 + 4 * 30000].reshape(-1, 4).astype(np.int64)
rec = rec[(rec[:, 0] >= t0) & (rec[:, 1] > 0)]
np.savez("gpurun_out/motion_items.npz", rec=rec, t0=t0, cta=tr)
print("per-item records saved to gpurun_out/motion_items.npz:", len(rec))
