"""Experiment: broadphase group size (codegen.GROUP_SIZE) vs kernel time.

    python scripts/exp_group.py [--sizes 2,3,4,5]
Motion config 2 (plan + rake) and configs 3 / 4 product-mode batches, L2
flushed before each launch; verdict words must not change with the group size.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import codegen, load_robot, runtime, workloads  # noqa: E402
from exp_variants import module_for  # noqa: E402

flush = None


def timed(fn, reps=20):
    ts = []
    for r in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.mean(ts))


def main():
    global flush
    p = argparse.ArgumentParser()
    p.add_argument("--sizes", default="2,3,4,5")
    a = p.parse_args()
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
    mw = workloads.config2()
    batch = {"cfg3": workloads.config3(), "cfg4": workloads.config4()}
    ref = {}
    for gs in [int(x) for x in a.sizes.split(",")]:
        codegen.GROUP_SIZE = gs
        rob = load_robot("arm7")
        mod = module_for(rob, 0)
        denv = runtime.DeviceEnv(mw.env.primitives)
        sd, gd = torch.from_numpy(mw.starts).cuda(), torch.from_numpy(mw.goals).cuda()
        ws = runtime.motion_workspace(len(sd))
        words = runtime.validate_motions_device(mod, denv, sd, gd, mw.resolution,
                                                workspace=ws)[0].cpu().numpy()
        assert np.array_equal(words, ref.setdefault("motion", words))
        us = timed(lambda: runtime.validate_motions_device(mod, denv, sd, gd, mw.resolution,
                                                           workspace=ws))
        line = [f"motion {us:6.1f}"]
        for key, wl in batch.items():
            m2 = module_for(load_robot(wl.robot), 0)
            de = runtime.DeviceEnv(wl.env.primitives)
            q = torch.from_numpy(wl.q).cuda()
            n = q.shape[1]
            out = runtime.validate_device(m2, de, q, n, n)
            w = out.cpu().numpy()
            assert np.array_equal(w, ref.setdefault(key, w))
            line.append(f"{key} {timed(lambda: runtime.validate_device(m2, de, q, n, n, out=out)):6.1f}")
        print(f"group {gs}: " + "  ".join(line), flush=True)


if __name__ == "__main__":
    main()
