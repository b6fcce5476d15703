"""The robots the benchmarks and tests use, as compiled ``KinematicProgram``s.

``data/robots.json`` holds each robot's program exactly as the REFERENCE's
tracing compiler emits it (vecmp.planners.build_robot, planners.py:59-68;
generated offline by scripts/make_robot_data.py and checked there against the
reference's program listings), plus its self-collision pairs, sphere model
and joint limits.  A caller of the drop-in passes its own reference-compiled
robot instead; the kernels only see the program and the pairs.

BASELINE.json names Panda, Fetch and Baxter workloads; those models are not
in the reference and are NOT reproduced here.  Per SURVEY.md
§8d the workloads use clearly labelled stand-ins:

* "panda"           -> ``arm7``, the reference's bundled 7-DoF arm (D = 7)
* ``fetch_standin`` -> SYNTHETIC: mobile base sphere + prismatic torso lift +
                       torso spheres + fixed mount + the arm7 chain (D = 8)
* ``baxter_standin``-> SYNTHETIC: pedestal + fixed torso + two arm7 chains
                       mounted at (0.05, +-0.25, 0.3), yaw +-0.785 (D = 14)
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from functools import lru_cache
from pathlib import Path

import numpy as np

from .program import KinematicProgram, program_from_record

DATA = Path(__file__).resolve().parent / "data" / "robots.json"

ROBOTS = ("arm7", "planar2", "fetch_standin", "baxter_standin")
#: BASELINE.json model name -> stand-in actually used
STANDIN_FOR = {"panda": "arm7", "fetch": "fetch_standin", "baxter": "baxter_standin"}


@dataclass(frozen=True)
class SelfCollisionPairs:
    """Unordered link-index pairs to test, as (lo, hi) tuples (the reference's
    pair-set type, robot.py:273-277)."""

    pairs: frozenset = field(default_factory=frozenset)


@dataclass(frozen=True)
class SphereModel:
    """Per-link fine spheres and coarse sphere, each ``(x, y, z, r)`` in the
    link frame (``None`` for unchecked links) - the data of the reference's
    sphere model (robot.py:189-203).  The kernels read radii and centres from
    the program; this travels with the robot for API parity."""

    fine: tuple
    coarse: tuple

    def checked_links(self) -> list[int]:
        return [i for i, spheres in enumerate(self.fine) if spheres]


@dataclass(frozen=True)
class Robot:
    """Compiled robot bundle (fields of the reference's planners.Robot,
    planners.py:48-56, without the URDF tree)."""

    model: SphereModel
    pairs: SelfCollisionPairs
    program: KinematicProgram
    limits: np.ndarray           # (dof, 2) float64
    name: str = "robot"
    links: tuple = ()
    source: str = ""

    @property
    def dof(self) -> int:
        return int(self.program.dof)


@lru_cache(maxsize=1)
def _records() -> dict:
    return json.loads(DATA.read_text())


def robot_from_record(rec: dict) -> Robot:
    prog = dict(rec["program"], dof=rec["dof"])
    sph = rec["spheres"]
    return Robot(
        model=SphereModel(fine=tuple(tuple(tuple(s) for s in link) for link in sph["fine"]),
                          coarse=tuple(None if s is None else tuple(s) for s in sph["coarse"])),
        pairs=SelfCollisionPairs(frozenset(tuple(p) for p in rec["pairs"])),
        program=program_from_record(prog),
        limits=np.asarray(rec["limits"], dtype=np.float64).reshape(-1, 2),
        name=rec["name"], links=tuple(rec["links"]), source=rec["source"])


def load_robot(name: str) -> Robot:
    """Bundled robot by name; BASELINE names map to their stand-ins."""
    return _load(STANDIN_FOR.get(name, name))


@lru_cache(maxsize=None)
def _load(name: str) -> Robot:
    recs = _records()
    if name not in recs:
        raise KeyError(f"unknown robot {name!r}; known: {ROBOTS}")
    return robot_from_record(recs[name])
