"""Generate golden fixtures from the REFERENCE implementation (run in the build
container only - /root/reference does not exist on the GPU box).

    python tests/golden/make_golden.py

Imports the reference package ``vecmp`` from /root/reference/pkg/src (and its
test helpers envgen.py / fk_reference.py) and records, for seeded inputs:

  programs.json  dump_program listings + self pairs of every robot the tests
                 use (reference program.py:217-244, robot.py:279-295)
  fk.npz         float32 marker centres streamed by evaluate_program
                 (program.py:157-214) and float64 centres from evaluate_graph
                 (trace.py:100-137)
  blocks.npz     validate_block verdicts at W = 8 (prune on / off), one wide
                 block, and reject_all per W = 8 block (collision.py:411-459)
  motion.npz     raked_motion_check (verdict, blocks) at W = 8 / 1 / 32,
                 forward and backward, plus discretization_count (motion.py)
  lanes.npz      l2_distance and discretization_count for D = 1..16
                 (lanes.py:106-113, motion.py:25-29)
  narrow.npz     sphere_vs_{sphere,capsule,cuboid}_lanes cases (collision.py:263-287)

Environments are stored as (kinds, params) arrays, see tests/golden_io.py.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import envgen  # noqa: E402  (reference test helper)
import fk_reference  # noqa: E402
import vecmp.collision as RC  # noqa: E402
from vecmp.lanes import ConfigBlock, l2_distance, soa_from_aos  # noqa: E402
from vecmp.motion import discretization_count, raked_motion_check  # noqa: E402
from vecmp.planners import build_robot  # noqa: E402
from vecmp.program import dump_program, evaluate_program  # noqa: E402
from vecmp.resources import environment_path  # noqa: E402
from vecmp.robot import load_sphere_model, parse_urdf  # noqa: E402
from vecmp.trace import evaluate_graph, optimize_graph, trace_kinematics  # noqa: E402

from golden_io import env_to_arrays  # noqa: E402
from paper_2309_14545_b200 import workloads  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "scripts"))
import make_robot_data  # noqa: E402  (URDF / sphere texts of the bundled robots)

ROBOTS = ("planar2", "arm7", "fetch_standin", "baxter_standin")


def ref_robot(name):
    urdf, spheres = make_robot_data.texts(name)
    tree = parse_urdf(urdf)
    model = load_sphere_model(tree, spheres)
    return tree, model, build_robot(tree, model)


def to_ref_env(env) -> RC.Environment:
    prims = []
    for p in env.primitives:
        if hasattr(p, "p0"):
            prims.append(RC.CapsuleObstacle(p0=np.asarray(p.p0, float), p1=np.asarray(p.p1, float),
                                            radius=float(p.radius)))
        elif hasattr(p, "half_extents"):
            prims.append(RC.BoxObstacle(center=np.asarray(p.center, float),
                                        half_extents=np.asarray(p.half_extents, float),
                                        rotation=np.asarray(p.rotation, float)))
        else:
            prims.append(RC.SphereObstacle(center=np.asarray(p.center, float),
                                           radius=float(p.radius)))
    return RC.Environment(primitives=prims, name=env.name)


def ctx(rob, env, width, prune=True):
    return RC.ValidationContext(program=rob.program, model=rob.model, pairs=rob.pairs, env=env,
                                width=width, prune=prune)


class Collect:
    def __init__(self):
        self.rows = []

    def __call__(self, marker, x, y, z):
        self.rows.append(np.stack([x, y, z]).copy())
        return False


# -------------------------------------------------------------------- parts

EXTRA_PROGRAMS = {
    "one_joint": ("""
<robot name="one"><link name="base"/><link name="arm"/>
<joint name="j" type="revolute"><parent link="base"/><child link="arm"/>
<axis xyz="0 0 1"/><limit lower="-3" upper="3"/></joint></robot>""",
                  "arm:\n  - {x: 0.5, y: 0.0, z: 0.0, r: 0.1}\n"),
    "skew_axis": ("""
<robot name="skew"><link name="a"/><link name="b"/><link name="c"/>
<joint name="j0" type="revolute"><parent link="a"/><child link="b"/>
<origin xyz="0.1 0.2 0.3" rpy="0.2 -0.4 0.5"/><axis xyz="1 1 0"/><limit lower="-2" upper="2"/></joint>
<joint name="j1" type="prismatic"><parent link="b"/><child link="c"/>
<origin xyz="0 0 0.4"/><axis xyz="0 0.6 0.8"/><limit lower="0" upper="0.5"/></joint></robot>""",
                  "b:\n  - {x: 0.1, y: 0.0, z: 0.0, r: 0.05}\n  - {x: 0.2, y: 0.1, z: 0.0, r: 0.04}\n"
                  "c:\n  - {x: 0.0, y: 0.0, z: 0.1, r: 0.03}\n"),
}


def programs() -> dict:
    out = {}
    for name in ROBOTS:
        _, _, rob = ref_robot(name)
        out[name] = {"dump": dump_program(rob.program),
                     "pairs": sorted([list(p) for p in rob.pairs.pairs])}
    for name, (urdf, spheres) in EXTRA_PROGRAMS.items():
        tree = parse_urdf(urdf)
        rob = build_robot(tree, load_sphere_model(tree, spheres))
        out[name] = {"dump": dump_program(rob.program),
                     "pairs": sorted([list(p) for p in rob.pairs.pairs]),
                     "urdf": urdf, "spheres": spheres}
    return out


def fk() -> dict:
    out = {}
    for name in ROBOTS:
        tree, model, rob = ref_robot(name)
        rng = np.random.default_rng(11)
        lims = rob.limits
        q = rng.uniform(lims[:, 0], lims[:, 1], size=(256, tree.dof)).astype(np.float32)
        q[0] = 0.0
        q[1] = lims[:, 0]
        q[2] = lims[:, 1]
        sink = Collect()
        evaluate_program(rob.program, ConfigBlock(dim=tree.dof, width=256,
                                                  data=np.ascontiguousarray(q.T), valid_count=256),
                         sink)
        f32 = np.stack(sink.rows)                       # (markers, 3, N)
        og = optimize_graph(trace_kinematics(tree, model))
        res = evaluate_graph(og, q.astype(np.float64))
        f64 = np.stack([res[(m.link, m.level, m.index)].T for m in rob.program.checks])
        # independent 4x4 chain oracle of the reference tests, first 16 configs
        chain = np.stack([np.stack([fk_reference.sphere_positions(tree, model, q[i])[
            (m.link, m.level, m.index)] for m in rob.program.checks]) for i in range(16)])
        out[f"q_{name}"] = np.ascontiguousarray(q.T)
        out[f"f32_{name}"] = f32
        out[f"f64_{name}"] = f64
        out[f"chain_{name}"] = chain                    # (16, markers, 3)
    return out


def scenes_for(name: str, rng) -> list:
    scale = {"planar2": 1.0, "arm7": 0.9, "fetch_standin": 1.0, "baxter_standin": 1.0}[name]
    envs = [envgen.random_environment(rng, scale) for _ in range(4)]
    if name == "planar2":
        for fname in ("wall_gap.yaml", "posts.yaml", "corridor.yaml"):
            envs.append(RC.load_environment(environment_path(fname).read_text()))
    elif name == "arm7":
        for fname in ("tabletop.yaml", "shelf.yaml", "cage.yaml"):
            envs.append(RC.load_environment(environment_path(fname).read_text()))
        envs.append(to_ref_env(workloads.config1(8).env))
        envs.append(to_ref_env(workloads.config2_scene()))
    elif name == "fetch_standin":
        envs.append(to_ref_env(workloads.config3(8).env))
    else:
        envs.append(to_ref_env(workloads.config4(8).env))
    return envs


def blocks() -> dict:
    out = {}
    for name in ROBOTS:
        tree, model, rob = ref_robot(name)
        rng = np.random.default_rng(23)
        lims = rob.limits
        n = 512
        q = rng.uniform(lims[:, 0], lims[:, 1], size=(n, tree.dof)).astype(np.float32)
        qs = np.ascontiguousarray(q.T)
        out[f"q_{name}"] = qs
        for e, env in enumerate(scenes_for(name, rng)):
            kinds, params = env_to_arrays(env)
            out[f"env_{name}_{e}_kinds"] = kinds
            out[f"env_{name}_{e}_params"] = params
            res = {}
            for prune in (True, False):
                c8 = ctx(rob, env, 8, prune)
                res[f"w8_p{int(prune)}"] = np.concatenate(
                    [c8.validate_block(soa_from_aos(list(q[i:i + 8]), width=8)) for i in range(0, n, 8)])
            wide = ctx(rob, env, n, True)
            res["wide"] = wide.validate_block(ConfigBlock(dim=tree.dof, width=n, data=qs, valid_count=n))
            c8 = ctx(rob, env, 8, True)
            res["reject_all"] = np.concatenate(
                [c8.validate_block(soa_from_aos(list(q[i:i + 8]), width=8), reject_all=True)
                 for i in range(0, n, 8)])
            for k, v in res.items():
                out[f"v_{name}_{e}_{k}"] = v.astype(bool)
    return out


def motion() -> dict:
    out = {}
    cases = []
    # planar2 over the reference's toy environments, short random steps like test_motion
    tree, model, rob = ref_robot("planar2")
    rng = np.random.default_rng(31)
    for e, fname in enumerate(("wall_gap.yaml", "posts.yaml", "corridor.yaml")):
        env = RC.load_environment(environment_path(fname).read_text())
        lims = rob.limits
        s = rng.uniform(lims[:, 0], lims[:, 1], size=(60, 2)).astype(np.float32)
        g = np.clip(s + rng.uniform(-0.7, 0.7, size=(60, 2)), lims[:, 0], lims[:, 1]).astype(np.float32)
        g[:10] = rng.uniform(lims[:, 0], lims[:, 1], size=(10, 2)).astype(np.float32)
        g[10] = s[10]                                       # zero-length motion
        cases.append(("planar2", e, env, s, g, 0.05))
    # arm7 over the config-2 scene, first 160 committed edges (half forced free)
    tree, model, rob = ref_robot("arm7")
    wl = workloads.config2()
    cases.append(("arm7", 0, to_ref_env(wl.env), wl.starts[:160], wl.goals[:160], wl.resolution))
    robots_cache = {}
    for robot, e, env, s, g, res in cases:
        if robot not in robots_cache:
            robots_cache[robot] = ref_robot(robot)[2]
        rob = robots_cache[robot]
        key = f"{robot}_{e}"
        kinds, params = env_to_arrays(env)
        out[f"env_{key}_kinds"], out[f"env_{key}_params"] = kinds, params
        out[f"starts_{key}"], out[f"goals_{key}"] = s, g
        out[f"res_{key}"] = np.float64(res)
        out[f"n_{key}"] = np.asarray([discretization_count(a, b, res) for a, b in zip(s, g)], np.int64)
        for width in (8, 1, 32):
            for backward in (False, True):
                c = ctx(rob, env, width)
                r = [raked_motion_check(a, b, c, res, backward=backward) for a, b in zip(s, g)]
                tag = f"{key}_w{width}_b{int(backward)}"
                out[f"verdict_{tag}"] = np.asarray([v for v, _ in r], bool)
                out[f"blocks_{tag}"] = np.asarray([k for _, k in r], np.int64)
    return out


def lanes() -> dict:
    rng = np.random.default_rng(41)
    out = {}
    for d in range(1, 17):
        a = rng.normal(size=(64, d)).astype(np.float32)
        b = rng.normal(size=(64, d)).astype(np.float32)
        a[0] = b[0]
        out[f"a_{d}"], out[f"b_{d}"] = a, b
        out[f"l2_{d}"] = np.asarray([l2_distance(x, y) for x, y in zip(a, b)], np.float64)
        for tag, res in (("r32", 1.0 / 32.0), ("r05", 0.05), ("r07", 0.07)):
            out[f"n_{tag}_{d}"] = np.asarray([discretization_count(x, y, res) for x, y in zip(a, b)],
                                             np.int64)
    return out


def narrow() -> dict:
    rng = np.random.default_rng(43)
    out = {}
    k = 1500
    # spheres
    c = rng.normal(size=(k, 3))
    r = rng.uniform(0.05, 0.5, size=k)
    pts = rng.normal(scale=1.5, size=(k, 8, 3)).astype(np.float32)
    rs = rng.uniform(0.05, 0.5, size=k)
    hits = np.stack([RC.sphere_vs_sphere_lanes(*pts[i].T, float(rs[i]),
                                               RC.SphereObstacle(center=c[i], radius=float(r[i])))
                     for i in range(k)])
    out.update(sph_c=c, sph_r=r, sph_pts=pts, sph_rs=rs, sph_hits=hits)
    # capsules (incl. degenerate)
    a = rng.normal(size=(k, 3))
    b = a + rng.normal(scale=0.8, size=(k, 3))
    b[:20] = a[:20]
    r = rng.uniform(0.05, 0.6, size=k)
    pts = rng.normal(scale=1.5, size=(k, 8, 3)).astype(np.float32)
    rs = rng.uniform(0.05, 0.5, size=k)
    hits = np.stack([RC.sphere_vs_capsule_lanes(*pts[i].T, float(rs[i]),
                                                RC.CapsuleObstacle(p0=a[i], p1=b[i], radius=float(r[i])))
                     for i in range(k)])
    out.update(cap_p0=a, cap_p1=b, cap_r=r, cap_pts=pts, cap_rs=rs, cap_hits=hits)
    # cuboids
    c = rng.normal(size=(k, 3))
    h = rng.uniform(0.1, 0.8, size=(k, 3))
    rot = np.stack([fk_reference.axis_angle(rng.normal(size=3), float(rng.uniform(0, np.pi)))
                    for _ in range(k)])
    pts = rng.normal(scale=1.5, size=(k, 8, 3)).astype(np.float32)
    rs = rng.uniform(0.05, 0.5, size=k)
    rs[:50] = rng.uniform(1.0, 2.0, size=50)            # large radii exercise the non-SAT path
    hits = np.stack([RC.sphere_vs_cuboid_lanes(*pts[i].T, float(rs[i]),
                                               RC.BoxObstacle(center=c[i], half_extents=h[i],
                                                              rotation=rot[i]))
                     for i in range(k)])
    out.update(box_c=c, box_h=h, box_rot=rot, box_pts=pts, box_rs=rs, box_hits=hits)
    return out


def prm_cases() -> dict:
    """Reference prm (planners.py:243-291) on the bundled problem sets."""
    import time
    from vecmp.planners import PlanningProblem, prm
    from vecmp.problems import load_problem_set
    from vecmp.resources import problem_set_path
    out = {}
    picks = (("toy_planar.yaml", "planar2", 3), ("arm_reach.yaml", "arm7", 2))
    for fname, robot, stride in picks:
        ps = load_problem_set(problem_set_path(fname))
        for case in ps.problems[::stride]:
            key = f"{robot}_{case.id}"
            t0 = time.perf_counter()
            res = prm(PlanningProblem(robot=ps.robot, env=case.env, start=case.start,
                                      goal=case.goal), ps.settings)
            dt = time.perf_counter() - t0
            kinds, params = env_to_arrays(case.env)
            out[f"env_{key}_kinds"], out[f"env_{key}_params"] = kinds, params
            out[f"start_{key}"], out[f"goal_{key}"] = case.start, case.goal
            s = ps.settings
            out[f"settings_{key}"] = np.asarray([s.resolution, s.max_iterations, s.prm_k,
                                                 s.prm_batch, float(s.rake_backward), s.width])
            out[f"iterations_{key}"] = np.int64(res.iterations)
            out[f"counters_{key}"] = np.asarray([res.blocks_evaluated, res.motion_checks], np.int64)
            out[f"seconds_{key}"] = np.float64(dt)
            out[f"path_{key}"] = (np.stack(res.path.waypoints) if res.success
                                  else np.zeros((0, len(case.start)), np.float32))
            print(f"  prm {key}: success={res.success} iterations={res.iterations} {dt:.2f} s")
    return out


def main() -> None:
    (HERE / "programs.json").write_text(json.dumps(programs(), indent=1, sort_keys=True) + "\n")
    if len(sys.argv) > 1 and sys.argv[1] == "prm":
        np.savez_compressed(HERE / "prm.npz", **prm_cases())
        return
    for name, fn in (("fk", fk), ("blocks", blocks), ("motion", motion), ("lanes", lanes),
                     ("narrow", narrow), ("prm", prm_cases)):
        np.savez_compressed(HERE / f"{name}.npz", **fn())
        print("wrote", name)


if __name__ == "__main__":
    main()
