import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads
torch.cuda.set_device(0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
def timed(fn, reps=15, doflush=True):
    ts = []
    for r in range(reps + 3):
        if doflush: flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if r >= 3: ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))
small = torch.empty(32, device="cuda")
print("empty torch kernel", timed(lambda: small.zero_()), "noflush", timed(lambda: small.zero_(), doflush=False))
wl = workloads.config1(65536)
rob = load_robot(wl.robot)
ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
for n in (32, 128, 4096, 65536):
    qd = runtime.to_device(np.ascontiguousarray(wl.q[:, :n]))
    out = runtime.validate_device(ctx.module, ctx.device_env, qd, n, n)
    for kw in (dict(split=False), dict(split=False, early_exit=False), dict(split=False, prune=False), dict(split=True)):
        f = lambda: runtime.validate_device(ctx.module, ctx.device_env, qd, n, n, out=out, **kw)
        print(n, kw, "flush", round(timed(f),1), "noflush", round(timed(f, doflush=False),1))
