"""Experiment: 128- vs 256-thread validate CTAs per staged environment size
(config-5 scenes, arm7, product and dense, 2^20 configurations, L2 flushed).

    VMP_EXP_WIDE=0|1 python scripts/exp_wide.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
rob = load_robot("arm7")
n = 1 << 20
q = torch.from_numpy(workloads.uniform_configs(rob.limits, n, 50)).cuda()
out = torch.empty(n // 32, dtype=torch.int32, device="cuda")


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.mean(ts))


for p in (128, 256, 512, 1024):
    env = workloads.config5_scene(p) if p in (128, 1024) else workloads.mixed_scene(
        500 + p, p // 2, p // 4, p - p // 2 - p // 4, workloads.BOX_CFG1, 0.55, f"s{p}")
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, env)
    prod = timed(lambda: ctx.validate_batch(q, out=out))
    w = out.clone()
    dense = timed(lambda: ctx.validate_batch(q, early_exit=False, out=out))
    assert torch.equal(w, out)
    print(f"P={p} env {ctx.device_env.bytes} B: product {prod:.3f} ms  dense {dense:.3f} ms", flush=True)
