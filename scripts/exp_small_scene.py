"""Experiment: dense vs broadphase kernels for sphere-only (and few-primitive)
scenes, to choose vmp_validate's small_scene rule from data.

    python scripts/exp_small_scene.py            (dense = the small-scene rule's choice)
    VMP_EXP_NO_SMALL=1 python scripts/exp_small_scene.py   (rule off: one-pass broadphase)
Prints per-batch ms (L2 flushed) for arm7 at 65,536 and 1,048,576 configurations.
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
qall = torch.from_numpy(workloads.uniform_configs(rob.limits, 1 << 20, 70)).cuda()


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


for ns, nc, nb in ((32, 0, 0), (64, 0, 0), (128, 0, 0), (256, 0, 0), (1024, 0, 0), (16, 8, 8),
                   (0, 4, 12)):
    env = workloads.mixed_scene(950 + ns, nb, nc, ns, workloads.BOX_CFG1, 0.45, f"s{ns}")
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, env)
    row = []
    for n in (1 << 16, 1 << 20):
        q = qall[:, :n]
        out = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
        auto = timed(lambda: runtime.validate_device(ctx.module, ctx.device_env, q, n, n, out=out,
                                                     split=False))
        dense = timed(lambda: runtime.validate_device(ctx.module, ctx.device_env, q, n, n, out=out,
                                                      split=False, early_exit=False))
        rate = 1 - runtime.unpack_bits(out.cpu().numpy(), n).mean()
        row.append(f"n={n}: auto {auto:.4f} ms dense {dense:.4f} ms (collision {rate:.2f})")
    print(f"spheres {ns} capsules {nc} boxes {nb}: " + " | ".join(row), flush=True)
