"""(De)serialisation of obstacle scenes for the golden fixtures.

kinds: int8 per primitive (0 sphere, 1 capsule, 2 cuboid)
params: float64 (K, 15) - sphere c(3) r; capsule p0(3) p1(3) r; cuboid c(3) h(3) R(9 row-major)
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def env_to_arrays(env):
    kinds, params = [], []
    for p in env.primitives:
        row = np.zeros(15)
        if hasattr(p, "p0"):
            kinds.append(1)
            row[0:3], row[3:6], row[6] = p.p0, p.p1, p.radius
        elif hasattr(p, "half_extents"):
            kinds.append(2)
            row[0:3], row[3:6], row[6:15] = p.center, p.half_extents, np.asarray(p.rotation).reshape(9)
        else:
            kinds.append(0)
            row[0:3], row[3] = p.center, p.radius
        params.append(row)
    return np.asarray(kinds, np.int8), np.asarray(params, np.float64).reshape(-1, 15)


def arrays_to_env(kinds, params, name="golden"):
    from paper_2309_14545_b200.collision import (BoxObstacle, CapsuleObstacle, Environment,
                                                 SphereObstacle)
    prims = []
    for k, row in zip(kinds, params):
        if k == 0:
            prims.append(SphereObstacle(center=row[0:3].copy(), radius=float(row[3])))
        elif k == 1:
            prims.append(CapsuleObstacle(p0=row[0:3].copy(), p1=row[3:6].copy(), radius=float(row[6])))
        else:
            prims.append(BoxObstacle(center=row[0:3].copy(), half_extents=row[3:6].copy(),
                                     rotation=row[6:15].reshape(3, 3).copy()))
    return Environment(primitives=prims, name=name)


def load(name: str):
    return np.load(GOLDEN / f"{name}.npz")


def env_from(fixture, prefix: str):
    return arrays_to_env(fixture[f"{prefix}_kinds"], fixture[f"{prefix}_params"], prefix)
