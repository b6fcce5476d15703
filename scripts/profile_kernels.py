"""Launch the hot kernels a few times for ncu captures (no timing printed).

    python scripts/profile_kernels.py motion|cfg1|cfg3|cfg4|cfg5_<P>|fk|knn [--reps 3] [--dense] [--n N]
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("what")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--dense", action="store_true")
    p.add_argument("--n", type=int, default=1 << 20)
    a = p.parse_args()
    torch.cuda.set_device(0)
    if a.what == "motion":
        mw = workloads.config2()
        rob = load_robot(mw.robot)
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
        sd, gd = torch.from_numpy(mw.starts).cuda(), torch.from_numpy(mw.goals).cuda()
        for _ in range(a.reps):
            runtime.validate_motions_device(ctx.module, ctx.device_env, sd, gd, mw.resolution)
    elif a.what == "knn":
        import numpy as np
        from paper_2309_14545_b200.nn import NNIndex
        rng = np.random.default_rng(0)
        idx = NNIndex(7)
        idx.insert_many(rng.uniform(-1, 1, size=(100_000, 7)), range(100_000))
        qs = rng.uniform(-1, 1, size=(4096, 7))
        for _ in range(a.reps):
            idx.k_nearest_many(qs, 8)
    elif a.what == "fk":
        wl = workloads.config3()
        rob = load_robot(wl.robot)
        q = torch.from_numpy(wl.q).cuda()
        for _ in range(a.reps):
            runtime.fk_spheres(rob.program, q)
    else:
        if a.what.startswith("cfg5_"):
            wl = workloads.config5(a.n, int(a.what[5:]))
        else:
            wl = {"cfg1": workloads.config1, "cfg3": workloads.config3,
                  "cfg4": workloads.config4}[a.what]()
        rob = load_robot(wl.robot)
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
        q = torch.from_numpy(wl.q).cuda()
        for _ in range(a.reps):
            ctx.validate_batch(q, early_exit=not a.dense)
    torch.cuda.synchronize()
    print("ok", a.what)


if __name__ == "__main__":
    main()
