"""Experiment: motion rake with / without the coarse per-link prune (precise
back-to-back timing, 200 launches per measurement)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads  # noqa: E402

torch.cuda.set_device(0)
mw = workloads.config2()
rob = load_robot(mw.robot)
ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
sd, gd = torch.from_numpy(mw.starts).cuda(), torch.from_numpy(mw.goals).cuda()
ws = runtime.motion_workspace(len(sd))
bits = torch.empty((len(sd) + 31) // 32, dtype=torch.int32, device="cuda")
ref = None
for rep in range(2):
    for prune in (True, False):
        b = runtime.validate_motions_device(ctx.module, ctx.device_env, sd, gd, mw.resolution,
                                            prune=prune, bits=bits, workspace=ws)[0].cpu().numpy()
        ref = b if ref is None else ref
        assert np.array_equal(b, ref)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(200):
            runtime.validate_motions_device(ctx.module, ctx.device_env, sd, gd, mw.resolution,
                                            prune=prune, bits=bits, workspace=ws)
        e.record()
        torch.cuda.synchronize()
        print(f"prune={prune}: {s.elapsed_time(e) * 1e3 / 200:.2f} us per call", flush=True)
