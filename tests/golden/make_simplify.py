"""Golden fixtures for the batched simplifier, from the REFERENCE (build container only).

    python tests/golden/make_simplify.py     -> tests/golden/simplify.npz

For problems of the bundled problem sets, the reference rrt_connect
(planners.py:180-210) produces a path; the reference shortcut, bspline_smooth
and simplify_path (simplify.py:61-118) are then run on it with the problem
set's resolution and recorded together with the input path, the environment
and the settings.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "tests"))

from vecmp.collision import ValidationContext  # noqa: E402
from vecmp.planners import PlanningProblem, rrt_connect  # noqa: E402
from vecmp.problems import load_problem_set  # noqa: E402
from vecmp.resources import problem_set_path  # noqa: E402
from vecmp.simplify import SimplifySettings, bspline_smooth, shortcut, simplify_path  # noqa: E402

from golden_io import env_to_arrays  # noqa: E402

PICKS = (("toy_planar.yaml", "planar2", 2, (0, 7)), ("arm_reach.yaml", "arm7", 1, (0, 3)))
#: long inputs: the first planned path of these sets re-sampled to LONG waypoints
#: with seeded zig-zag noise on the interior ones (exercises multi-window smoothing
#: and many shortcut rounds)
LONG = (("toy_planar.yaml", "planar2", 0.05), ("arm_reach.yaml", "arm7", 0.03))
LONG_WAYPOINTS = 80


def long_path(waypoints, noise, seed):
    wps = np.stack(waypoints).astype(np.float64)
    seg = np.linalg.norm(np.diff(wps, axis=0), axis=1)
    cum = np.concatenate([[0.0], np.cumsum(seg)])
    u = np.linspace(0.0, cum[-1], LONG_WAYPOINTS)
    out = np.stack([np.interp(u, cum, wps[:, j]) for j in range(wps.shape[1])], axis=1)
    rng = np.random.default_rng(seed)
    out[1:-1] += rng.uniform(-noise, noise, size=out[1:-1].shape)
    out = out.astype(np.float32)
    out[0], out[-1] = waypoints[0], waypoints[-1]
    return list(out)


def main() -> None:
    out = {}
    cases = []                                          # (key, problem set, case, path, seed)
    for fname, robot, stride, seeds in PICKS:
        ps = load_problem_set(problem_set_path(fname))
        for case in ps.problems[::stride]:
            res = rrt_connect(PlanningProblem(robot=ps.robot, env=case.env, start=case.start,
                                              goal=case.goal), ps.settings)
            if not res.success or len(res.path.waypoints) < 3:
                continue
            for seed in seeds:
                cases.append((f"{robot}_{case.id}_s{seed}", ps, case, res.path, seed))
    for fname, robot, noise in LONG:
        ps = load_problem_set(problem_set_path(fname))
        case = ps.problems[0]
        res = rrt_connect(PlanningProblem(robot=ps.robot, env=case.env, start=case.start,
                                          goal=case.goal), ps.settings)
        path = type(res.path)(long_path(res.path.waypoints, noise, 5))
        cases.append((f"{robot}_long_s0", ps, case, path, 0))
    for key, ps, case, path, seed in cases:
        st = SimplifySettings(resolution=ps.settings.resolution, rng_seed=seed)
        ctx = ValidationContext(ps.robot.program, ps.robot.model, ps.robot.pairs, case.env,
                                width=ps.settings.width)
        counters = []

        def tally():
            counters.extend([ctx.motion_checks, ctx.blocks_evaluated])
            ctx.motion_checks = ctx.blocks_evaluated = 0
        t0 = time.perf_counter()
        sc = shortcut(path, ctx, st)
        tally()
        t1 = time.perf_counter()
        sm = bspline_smooth(path, ctx, st)
        tally()
        t2 = time.perf_counter()
        both = simplify_path(path, ctx, st)
        tally()
        kinds, params = env_to_arrays(case.env)
        out[f"env_{key}_kinds"], out[f"env_{key}_params"] = kinds, params
        out[f"settings_{key}"] = np.asarray([st.resolution, st.shortcut_attempts,
                                             st.smooth_rounds, st.rng_seed])
        out[f"path_{key}"] = np.stack(path.waypoints)
        out[f"shortcut_{key}"] = np.stack(sc.waypoints)
        out[f"smooth_{key}"] = np.stack(sm.waypoints)
        out[f"simplify_{key}"] = np.stack(both.waypoints)
        out[f"seconds_{key}"] = np.asarray([t1 - t0, t2 - t1])
        # ValidationContext counters (motion_checks, blocks_evaluated) of each
        # call: shortcut, bspline_smooth, simplify_path
        out[f"counters_{key}"] = np.asarray(counters, dtype=np.int64)
        out[f"width_{key}"] = np.asarray(ctx.width)
        print(f"{key}: {len(path.waypoints)} -> shortcut {len(sc.waypoints)} "
              f"({t1 - t0:.2f} s), smooth ({t2 - t1:.2f} s), "
              f"cost {path.cost:.3f} -> {both.cost:.3f}", flush=True)
    np.savez_compressed(HERE / "simplify.npz", **out)


if __name__ == "__main__":
    main()
