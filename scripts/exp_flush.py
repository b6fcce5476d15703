"""Experiment: config-2 step time with and without an L2 flush before each step
(how much of the step is cold-cache code/data fetch)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, workloads  # noqa: E402
from paper_2309_14545_b200 import motion as M  # noqa: E402

torch.cuda.set_device(0)
mw = workloads.config2()
rob = load_robot(mw.robot)
import os  # noqa: E402
# VMP_EXP_PRUNE=0: contexts without the coarse per-link prune (verdict-neutral)
ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env,
                        prune=os.environ.get("VMP_EXP_PRUNE", "1") != "0")
mv = M.MotionValidator(ctx, len(mw.starts), mw.resolution, width=32)
mv(mw.starts, mw.goals)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
small = torch.empty(1 << 10, dtype=torch.float32, device="cuda")
for mode in ("flush", "noflush", "flush", "noflush"):
    ts = []
    for _ in range(30):
        (flush if mode == "flush" else small).zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mv()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"{mode}: median {np.median(ts):.1f} us  min {np.min(ts):.1f} us")

# precise: 200 back-to-back replays between two events (event ticks are 2 us)
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200):
        mv()
    b.record()
    torch.cuda.synchronize()
    print(f"200 back-to-back replays: {a.elapsed_time(b) * 1e3 / 200:.2f} us per step")
