"""Motion rake throughput vs batch size: config-2 edges tiled to 4K .. 1M edges
(round 0 of one to hundreds of waves per warp), L2 flushed per launch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
mw = workloads.config2()
rob = load_robot(mw.robot)
ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
for tiles in (1, 2, 16, 64, 256):
    s = torch.from_numpy(np.tile(mw.starts, (tiles, 1))).cuda()
    g = torch.from_numpy(np.tile(mw.goals, (tiles, 1))).cuda()
    e = len(s)
    ws = runtime.motion_workspace(e)
    bits = torch.empty((e + 31) // 32, dtype=torch.int32, device="cuda")
    run = lambda: runtime.validate_motions_device(ctx.module, ctx.device_env, s, g, mw.resolution,
                                                  bits=bits, workspace=ws)
    run()
    ts = []
    for r in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b) / 1e3)
    t = float(np.mean(ts))
    print(f"E={e:8d}: {t * 1e3:.3f} ms, {e / t / 1e6:.1f} M edges/s", flush=True)
