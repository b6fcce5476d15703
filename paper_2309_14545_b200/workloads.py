"""Seeded synthetic workloads for BASELINE.json configs 1-5.

The paper measures on MotionBenchMaker scenes with the real Panda / Fetch /
Baxter models; none of those exist in the reference, so every workload here
is synthetic: labelled stand-in robots (robots.py) and seeded obstacle
scenes with the BASELINE distributions.  All random draws are
``np.random.default_rng(seed)`` in float64, cast to float32 where the path
consumes float32.

Scenes get the keep-out rule of SURVEY.md §8d: an obstacle's bounding sphere
must lie outside a vertical cylinder of radius ``keepout`` about the robot
base axis (otherwise nearly every state collides and the benchmark
degenerates to first-check exits).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .collision import BoxObstacle, CapsuleObstacle, Environment, SphereObstacle

BOX_CFG1 = ((-0.8, 0.8), (-0.8, 0.8), (0.0, 1.2))
BOX_CFG3 = ((-0.2, 1.4), (-0.8, 0.8), (0.0, 1.6))

#: keep-out radii (m) per robot, SURVEY.md §8d (arm7 0.3, fetch 0.4, baxter 0.5)
KEEPOUT = {"arm7": 0.3, "fetch_standin": 0.4, "baxter_standin": 0.5}


def _centre(rng, box) -> np.ndarray:
    return np.array([rng.uniform(lo, hi) for lo, hi in box])


def _unit(rng) -> np.ndarray:
    v = rng.normal(size=3)
    return v / np.linalg.norm(v)


def quat_to_matrix(q) -> np.ndarray:
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def _outside(centre, bound: float, keepout: float) -> bool:
    return float(np.hypot(centre[0], centre[1])) - bound >= keepout


def random_cuboid(rng, box, keepout: float) -> BoxObstacle:
    while True:
        c = _centre(rng, box)
        h = rng.uniform(0.02, 0.3, size=3)
        rot = quat_to_matrix(rng.normal(size=4))
        if _outside(c, float(np.linalg.norm(h)), keepout):
            return BoxObstacle(center=c, half_extents=h, rotation=rot)


def random_capsule(rng, box, keepout: float) -> CapsuleObstacle:
    while True:
        c = _centre(rng, box)
        r = rng.uniform(0.02, 0.08)
        length = rng.uniform(0.1, 0.6)
        axis = _unit(rng)
        if _outside(c, 0.5 * length + r, keepout):
            return CapsuleObstacle(p0=c - 0.5 * length * axis, p1=c + 0.5 * length * axis, radius=r)


def random_sphere(rng, box, keepout: float) -> SphereObstacle:
    while True:
        c = _centre(rng, box)
        r = rng.uniform(0.05, 0.15)
        if _outside(c, r, keepout):
            return SphereObstacle(center=c, radius=r)


def mixed_scene(seed: int, n_box: int, n_cap: int, n_sph: int, box=BOX_CFG1,
                keepout: float = 0.0, name: str = "scene") -> Environment:
    rng = np.random.default_rng(seed)
    prims = [random_cuboid(rng, box, keepout) for _ in range(n_box)]
    prims += [random_capsule(rng, box, keepout) for _ in range(n_cap)]
    prims += [random_sphere(rng, box, keepout) for _ in range(n_sph)]
    return Environment(primitives=prims, name=name)


def uniform_configs(limits: np.ndarray, n: int, seed: int) -> np.ndarray:
    """(dof, n) float32 SoA batch, uniform within joint limits."""
    rng = np.random.default_rng(seed)
    q = rng.uniform(limits[:, 0], limits[:, 1], size=(n, limits.shape[0]))
    return np.ascontiguousarray(q.T.astype(np.float32))


@dataclass
class BatchWorkload:
    name: str
    robot: str
    q: np.ndarray          # (dof, N) float32
    env: Environment
    note: str


def config1(n: int = 65536) -> BatchWorkload:
    """Panda(arm7) 65,536 configs, 32 spheres r~U[.05,.15] in [-.8,.8]^2 x [0,1.2]."""
    from .robots import load_robot
    rob = load_robot("arm7")
    rng = np.random.default_rng(1)
    prims = [SphereObstacle(center=_centre(rng, BOX_CFG1), radius=rng.uniform(0.05, 0.15))
             for _ in range(32)]
    return BatchWorkload("cfg1_arm7_32spheres", "arm7", uniform_configs(rob.limits, n, 0),
                         Environment(prims, "cfg1"), "seed 0 configs, seed 1 scene, no keep-out")


def config3(n: int = 1 << 20) -> BatchWorkload:
    from .robots import load_robot
    rob = load_robot("fetch_standin")
    env = mixed_scene(3, 32, 16, 16, BOX_CFG3, KEEPOUT["fetch_standin"], "cfg3")
    return BatchWorkload("cfg3_fetch_standin_64mixed", "fetch_standin",
                         uniform_configs(rob.limits, n, 30), env,
                         "32 cuboids + 16 cylinders(capsules) + 16 spheres, keep-out 0.4 m")


def config4(n: int = 1 << 20) -> BatchWorkload:
    from .robots import load_robot
    rob = load_robot("baxter_standin")
    env = mixed_scene(4, 48, 16, 0, BOX_CFG3, KEEPOUT["baxter_standin"], "cfg4")
    table = BoxObstacle(center=np.array([0.9, 0.0, 0.7]), half_extents=np.array([0.5, 0.3, 0.025]),
                        rotation=np.eye(3))
    env.primitives.append(table)
    return BatchWorkload("cfg4_baxter_standin_65", "baxter_standin",
                         uniform_configs(rob.limits, n, 40), env,
                         "48 cuboids + 16 cylinders + table (x=0.9, z=0.7), keep-out 0.5 m")


#: keep-out per obstacle count for the config-5 sweep (rate kept in 20-60 %)
SWEEP_KEEPOUT = {16: 0.1, 128: 0.45, 1024: 0.6}


def config5_scene(p: int) -> Environment:
    kb, kc = p // 2, p // 4
    return mixed_scene(500 + p, kb, kc, p - kb - kc, BOX_CFG1, SWEEP_KEEPOUT.get(p, 0.5), f"cfg5_{p}")


def config5(n: int, p: int) -> BatchWorkload:
    from .robots import load_robot
    rob = load_robot("arm7")
    return BatchWorkload(f"cfg5_arm7_P{p}_N{n}", "arm7", uniform_configs(rob.limits, n, 50),
                         config5_scene(p), f"{p} mixed primitives (50% cuboid/25% capsule/25% sphere)")


def config2_scene() -> Environment:
    return mixed_scene(2, 24, 8, 0, BOX_CFG1, KEEPOUT["arm7"], "cfg2")


CFG2_RESOLUTION = 1.0 / 32.0


@dataclass
class MotionWorkload:
    name: str
    robot: str
    starts: np.ndarray     # (E, dof) float32
    goals: np.ndarray
    env: Environment
    resolution: float
    note: str


def config2() -> MotionWorkload:
    """Panda(arm7) 4,096 edges, even-indexed forced free (tests/golden/make_workloads.py)."""
    from pathlib import Path
    data = np.load(Path(__file__).resolve().parent / "data" / "cfg2_edges.npz")
    return MotionWorkload("cfg2_arm7_4096edges_24box_8cap", "arm7",
                          np.ascontiguousarray(data["starts"]), np.ascontiguousarray(data["goals"]),
                          config2_scene(), float(data["resolution"]),
                          "24 cuboids + 8 capsules, keep-out 0.3 m, resolution 1/32, "
                          "even edges forced free")
