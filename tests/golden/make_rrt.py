"""Golden runs of the REFERENCE rrt_connect (planners.py:180-210) on the
bundled problem sets (build container only).

    python tests/golden/make_rrt.py     -> tests/golden/rrt.npz

Records, per problem: environment, start, goal, planner settings, the
returned waypoints, iteration count, the ValidationContext counters
(blocks_evaluated, motion_checks) and the reference's wall time.
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

from vecmp.planners import PlanningProblem, rrt_connect  # noqa: E402
from vecmp.problems import load_problem_set  # noqa: E402
from vecmp.resources import problem_set_path  # noqa: E402

from golden_io import env_to_arrays  # noqa: E402
from vecmp.planners import PlannerSettings  # noqa: E402

PICKS = (("toy_planar.yaml", "planar2"), ("arm_reach.yaml", "arm7"))
#: stress cases: arm7 in the config-2 clutter (24 cuboids + 8 capsules) between
#: the endpoints of the first CLUTTER_COUNT odd config-2 edges with both
#: endpoints free (odd edges are not forced free; most collide)
CLUTTER_COUNT = 4
CLUTTER = PlannerSettings(resolution=1.0 / 32.0, range=0.5, max_iterations=3000)


def clutter_cases():
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(HERE))
    from make_golden import ref_robot, to_ref_env
    from paper_2309_14545_b200 import workloads
    from vecmp.collision import ValidationContext
    mw = workloads.config2()
    _, _, robot = ref_robot("arm7")
    env = to_ref_env(mw.env)
    ctx = ValidationContext(robot.program, robot.model, robot.pairs, env)
    found = 0
    for e in range(1, len(mw.starts), 2):
        if found == CLUTTER_COUNT:
            break
        if ctx.state_valid(mw.starts[e]) and ctx.state_valid(mw.goals[e]):
            found += 1
            yield f"arm7_clutter_{e}", robot, env, mw.env, mw.starts[e], mw.goals[e], CLUTTER


def main() -> None:
    out = {}
    for fname, robot in PICKS:
        ps = load_problem_set(problem_set_path(fname))
        for case in ps.problems:
            key = f"{robot}_{case.id}"
            t0 = time.perf_counter()
            res = rrt_connect(PlanningProblem(robot=ps.robot, env=case.env, start=case.start,
                                              goal=case.goal), ps.settings)
            dt = time.perf_counter() - t0
            s = ps.settings
            kinds, params = env_to_arrays(case.env)
            out[f"env_{key}_kinds"], out[f"env_{key}_params"] = kinds, params
            out[f"start_{key}"], out[f"goal_{key}"] = case.start, case.goal
            out[f"settings_{key}"] = np.asarray([s.resolution, s.range, s.max_iterations,
                                                 float(s.rake_backward), s.width])
            out[f"iterations_{key}"] = np.int64(res.iterations)
            out[f"counters_{key}"] = np.asarray([res.blocks_evaluated, res.motion_checks], np.int64)
            out[f"seconds_{key}"] = np.float64(dt)
            out[f"path_{key}"] = (np.stack(res.path.waypoints) if res.success
                                  else np.zeros((0, len(case.start)), np.float32))
            print(f"rrt {key}: success={res.success} iterations={res.iterations} "
                  f"waypoints={len(res.path.waypoints) if res.success else 0} "
                  f"checks={res.motion_checks} {dt:.2f} s", flush=True)
    for key, robot, env, my_env, start, goal, s in clutter_cases():
        t0 = time.perf_counter()
        res = rrt_connect(PlanningProblem(robot=robot, env=env, start=start, goal=goal), s)
        dt = time.perf_counter() - t0
        kinds, params = env_to_arrays(my_env)
        out[f"env_{key}_kinds"], out[f"env_{key}_params"] = kinds, params
        out[f"start_{key}"], out[f"goal_{key}"] = start, goal
        out[f"settings_{key}"] = np.asarray([s.resolution, s.range, s.max_iterations,
                                             float(s.rake_backward), s.width])
        out[f"iterations_{key}"] = np.int64(res.iterations)
        out[f"counters_{key}"] = np.asarray([res.blocks_evaluated, res.motion_checks], np.int64)
        out[f"seconds_{key}"] = np.float64(dt)
        out[f"path_{key}"] = (np.stack(res.path.waypoints) if res.success
                              else np.zeros((0, len(start)), np.float32))
        print(f"rrt {key}: success={res.success} iterations={res.iterations} "
              f"waypoints={len(res.path.waypoints) if res.success else 0} "
              f"checks={res.motion_checks} {dt:.2f} s", flush=True)
    np.savez_compressed(HERE / "rrt.npz", **out)


if __name__ == "__main__":
    main()
