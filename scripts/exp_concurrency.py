"""Experiment: do two independent config-2 rakes (separate MotionValidators,
separate streams) overlap on the GPU?  Compares 100 alternating graph replays
on one stream with the same replays spread over two streams.

    python scripts/exp_concurrency.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, workloads  # noqa: E402
from paper_2309_14545_b200 import motion as M  # noqa: E402

torch.cuda.set_device(0)
mw = workloads.config2()
rob = load_robot(mw.robot)
ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
mvs = [M.MotionValidator(ctx, len(mw.starts), mw.resolution) for _ in range(2)]
for mv in mvs:
    mv(mw.starts, mw.goals)
torch.cuda.synchronize()
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
N = 100
for mode in ("one stream", "two streams", "one stream", "two streams"):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in streams:
        s.wait_event(a)
    for i in range(N):
        st = streams[i % 2] if mode == "two streams" else streams[0]
        with torch.cuda.stream(st):
            mvs[i % 2]()
    for s in streams:
        b.wait_stream(s) if hasattr(b, "wait_stream") else None
    torch.cuda.current_stream().wait_stream(streams[0])
    torch.cuda.current_stream().wait_stream(streams[1])
    b.record()
    torch.cuda.synchronize()
    print(f"{mode}: {a.elapsed_time(b) * 1e3 / N:.1f} us per rake")
