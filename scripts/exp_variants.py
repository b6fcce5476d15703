"""Experiment: time codegen variants (launch bounds, prune) on the GPU.

    python scripts/exp_variants.py [--min-blocks 0,6,8]
Prints one line per (workload, variant) with the median kernel time.
"""

import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import codegen, load_robot, runtime, workloads  # noqa: E402
from paper_2309_14545_b200._native import RobotDesc, check, lib  # noqa: E402


def module_for(rob, min_blocks: int):
    src = codegen.generate_source(rob.program, rob.pairs)
    if min_blocks:
        for k in ("vmp_motion", "vmp_validate"):
            src = src.replace(f"__launch_bounds__({codegen.BLOCK}) {k}",
                              f"__launch_bounds__({codegen.BLOCK}, {min_blocks}) {k}")
    path = runtime.compile_cubin(src, "exp")
    mod = runtime.RobotModule.__new__(runtime.RobotModule)
    desc = RobotDesc(int(rob.program.dof), len(rob.program.kinds), len(rob.program.checks), 1)
    h = ctypes.c_void_p()
    check(lib().vmp_robot_load(str(path).encode(), ctypes.byref(desc), ctypes.byref(h)))
    mod.handle, mod.dof = h, int(rob.program.dof)
    mod.n_ops, mod.n_markers = len(rob.program.kinds), len(rob.program.checks)
    return mod


def time_it(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--min-blocks", default="0,6,8")
    a = p.parse_args()
    torch.cuda.set_device(0)
    mw = workloads.config2()
    batch = {"cfg1": workloads.config1(), "cfg3": workloads.config3(), "cfg4": workloads.config4()}
    for mb in [int(x) for x in a.min_blocks.split(",")]:
        rob = load_robot("arm7")
        mod = module_for(rob, mb)
        denv = runtime.DeviceEnv(mw.env.primitives)
        sd, gd = torch.from_numpy(mw.starts).cuda(), torch.from_numpy(mw.goals).cuda()
        ws = runtime.motion_workspace(len(sd))
        for prune in (True, False):
            ms = time_it(lambda: runtime.validate_motions_device(mod, denv, sd, gd, mw.resolution,
                                                                 prune=prune, workspace=ws))
            print(f"motion cfg2 minblocks={mb} prune={prune}: {ms * 1e3:.1f} us", flush=True)
        for key, wl in batch.items():
            rob = load_robot(wl.robot)
            m2 = mod if wl.robot == "arm7" else module_for(rob, mb)
            de = runtime.DeviceEnv(wl.env.primitives)
            q = torch.from_numpy(wl.q).cuda()
            n = q.shape[1]
            for prune in (True, False):
                for early in (True, False):
                    ms = time_it(lambda: runtime.validate_device(m2, de, q, n, n, prune=prune,
                                                                 early_exit=early))
                    print(f"{key} minblocks={mb} prune={prune} early={early}: {ms * 1e3:.1f} us",
                          flush=True)


if __name__ == "__main__":
    main()
