"""Test helpers that derive new robots / scenes from existing ones.

``translate_program`` moves a robot rigidly: every sphere-centre op of a
``KinematicProgram`` gets a constant offset added (constant centres are
folded), the result is again a straight-line program the reference's
interpreter (and the oracle restating it) evaluates as-is.  Used by the
translated-scene parity tests (robot base and obstacles shifted
by 5, 10 and 30 m).
"""

from __future__ import annotations

import numpy as np

from paper_2309_14545_b200.collision import (BoxObstacle, CapsuleObstacle, Environment,
                                             SphereObstacle)
from paper_2309_14545_b200.program import CheckMarker, KinematicProgram

CONST, ADD = 0, 2


def translate_program(program, offset) -> KinematicProgram:
    kinds = [int(k) for k in program.kinds]
    a = [int(x) for x in program.a]
    b = [int(x) for x in program.b]
    values = [float(v) for v in program.values]
    off_op = {}
    for axis in range(3):                       # one CONST op per axis offset
        off_op[axis] = len(kinds)
        kinds.append(CONST)
        a.append(-1)
        b.append(-1)
        values.append(float(offset[axis]))
    moved: dict[tuple, int] = {}

    def shift(op: int, axis: int) -> int:
        key = (op, axis)
        if key not in moved:
            moved[key] = len(kinds)
            if kinds[op] == CONST:              # constant centre stays constant
                kinds.append(CONST)
                a.append(-1)
                b.append(-1)
                values.append(float(np.float32(values[op]) + np.float64(offset[axis])))
            else:
                kinds.append(ADD)
                a.append(op)
                b.append(off_op[axis])
                values.append(0.0)
        return moved[key]

    checks = []
    for m in program.checks:
        xyz = tuple(shift(int(v), axis) for axis, v in enumerate(m.xyz))
        checks.append(CheckMarker(link=m.link, level=m.level, index=m.index, radius=m.radius,
                                  xyz=xyz, position=max(xyz) + 1))
    return KinematicProgram(dof=int(program.dof), kinds=np.asarray(kinds, np.int8),
                            a=np.asarray(a, np.int32), b=np.asarray(b, np.int32),
                            values=np.asarray(values, np.float64), checks=checks,
                            outputs={})


def translate_env(env, offset) -> Environment:
    off = np.asarray(offset, np.float64)
    prims = []
    for p in env.primitives:
        if hasattr(p, "p0"):
            prims.append(CapsuleObstacle(p0=np.asarray(p.p0) + off, p1=np.asarray(p.p1) + off,
                                         radius=p.radius))
        elif hasattr(p, "half_extents"):
            prims.append(BoxObstacle(center=np.asarray(p.center) + off,
                                     half_extents=np.asarray(p.half_extents),
                                     rotation=np.asarray(p.rotation)))
        else:
            prims.append(SphereObstacle(center=np.asarray(p.center) + off, radius=p.radius))
    return Environment(primitives=prims, name=f"{env.name}+{tuple(np.round(off, 3))}")
