"""Experiment: simplest per-slot-stream pipeline (H2D, graph replay, D2H all on
the slot's own stream; the host waits only for the batch `depth` steps back)
vs MotionPipeline, e2e per step.

    python scripts/exp_pipe2.py [--steps 100]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads  # noqa: E402
from paper_2309_14545_b200 import motion as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=100)
a = p.parse_args()
torch.cuda.set_device(0)
mw = workloads.config2()
rob = load_robot(mw.robot)
ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
E = len(mw.starts)
hs = torch.from_numpy(mw.starts).pin_memory()
hg = torch.from_numpy(mw.goals).pin_memory()
for depth in (4, 6, 8, 4, 6, 8):
    slots = [M.MotionValidator(ctx, E, mw.resolution, overlapped=True) for _ in range(depth)]
    streams = [torch.cuda.Stream() for _ in range(depth)]
    host = [torch.empty(s.bits.shape, dtype=torch.int32).pin_memory() for s in slots]
    done = [torch.cuda.Event() for _ in range(depth)]
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in streams:
        s.wait_event(t0)
    for i in range(a.steps):
        k = i % depth
        if i >= depth:
            done[k].synchronize()              # this slot's previous batch is on the host
        with torch.cuda.stream(streams[k]):
            slots[k].starts.copy_(hs, non_blocking=True)
            slots[k].goals.copy_(hg, non_blocking=True)
            slots[k]()
            host[k].copy_(slots[k].bits, non_blocking=True)
            done[k].record(streams[k])
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.steps
    ok = runtime.unpack_bits(host[0].numpy(), E).sum()
    print(f"per-slot streams, depth {depth}: {ms * 1e3:.1f} us per step, {E / ms / 1e3:.1f} M edges/s "
          f"({ok} valid)")
