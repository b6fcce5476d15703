"""Robot descriptions used by the benchmarks and tests.

``arm7`` and ``planar2`` restate, as compact tables, the two robots bundled
with the reference (pkg/src/vecmp/resources/robots/*.urdf, *_spheres.yaml):
the generated URDF/YAML text is not byte-identical to the reference files,
but it compiles to the identical KinematicProgram (tests/golden/programs.json).

BASELINE.json names Panda, Fetch and Baxter workloads; those models are not
in the reference and are NOT reproduced here.  Per SURVEY.md
§8d the workloads use clearly labelled SYNTHETIC STAND-INS:

* "panda"           -> ``arm7`` as-is (D = 7)
* ``fetch_standin`` -> mobile base sphere + prismatic torso lift + torso
                       spheres + fixed mount + the arm7 chain (D = 8)
* ``baxter_standin``-> pedestal + fixed torso + two arm7 chains mounted at
                       (0.05, +-0.25, 0.3) with yaw +-0.785 (D = 14)
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .program import KinematicProgram, schedule_program
from .robot import (KinematicTree, SelfCollisionPairs, SphereModel, default_self_collision_pairs,
                    load_sphere_model, parse_urdf)
from .trace import optimize_graph, trace_kinematics

# (name, kind, parent, child, xyz, rpy, axis, (lo, hi) or None)
_ARM7_JOINTS = (
    ("j1_pan", "revolute", "base_link", "shoulder_link", (0, 0, 0.20), "z", (-2.9, 2.9)),
    ("j2_lift", "revolute", "shoulder_link", "upper_link", (0, 0, 0.10), "y", (-1.9, 1.9)),
    ("j3_roll", "revolute", "upper_link", "elbow_link", (0, 0, 0.25), "z", (-2.9, 2.9)),
    ("j4_elbow", "revolute", "elbow_link", "forearm_link", (0, 0, 0.10), "y", (-2.2, 2.2)),
    ("j5_roll", "revolute", "forearm_link", "roll_link", (0, 0, 0.25), "z", (-2.9, 2.9)),
    ("j6_pitch", "revolute", "roll_link", "wrist_link", (0, 0, 0.10), "y", (-2.0, 2.0)),
    ("j7_spin", "continuous", "wrist_link", "hand_link", (0, 0, 0.10), "z", None),
    ("flange_mount", "fixed", "hand_link", "flange_link", (0, 0, 0.08), None, None),
    ("tool_mount", "fixed", "flange_link", "tool_link", (0, 0, 0.05), None, None),
)
_ARM7_LINKS = ("base_link", "shoulder_link", "upper_link", "elbow_link", "forearm_link",
               "roll_link", "wrist_link", "hand_link", "flange_link", "tool_link")
# link -> [(x, y, z, r)]
_ARM7_SPHERES = {
    "base_link": [(0, 0, 0.08, 0.11)],
    "shoulder_link": [(0, 0, 0.05, 0.08)],
    "upper_link": [(0, 0, 0.07, 0.075), (0, 0, 0.18, 0.07)],
    "elbow_link": [(0, 0, 0.05, 0.07)],
    "forearm_link": [(0, 0, 0.07, 0.065), (0, 0, 0.18, 0.06)],
    "roll_link": [(0, 0, 0.05, 0.06)],
    "wrist_link": [(0, 0, 0.05, 0.055)],
    "hand_link": [(0, 0, 0.04, 0.05)],
    "tool_link": [(0, 0, 0.02, 0.045)],
}

_PLANAR2_LINKS = ("base_link", "upper_link", "fore_link", "tool_link")
_PLANAR2_JOINTS = (
    ("shoulder", "revolute", "base_link", "upper_link", (0, 0, 0), "z", (-3.1, 3.1)),
    ("elbow", "revolute", "upper_link", "fore_link", (0.5, 0, 0), "z", (-2.9, 2.9)),
    ("tool_mount", "fixed", "fore_link", "tool_link", (0.5, 0, 0), None, None),
)
_PLANAR2_SPHERES = {
    "upper_link": [(0.15, 0, 0, 0.08), (0.35, 0, 0, 0.08)],
    "fore_link": [(0.15, 0, 0, 0.08), (0.35, 0, 0, 0.08)],
    "tool_link": [(0, 0, 0, 0.06)],
}

_AXES = {"x": "1 0 0", "y": "0 1 0", "z": "0 0 1"}


def _fmt(v) -> str:
    return " ".join(repr(float(x)) for x in v)


def _urdf(name: str, links, joints) -> str:
    out = [f'<robot name="{name}">']
    out += [f'  <link name="{ln}"/>' for ln in links]
    for jn, kind, parent, child, xyz, *rest in joints:
        axis, limits = rest[0], rest[1]
        rpy = rest[2] if len(rest) > 2 else (0, 0, 0)
        out.append(f'  <joint name="{jn}" type="{kind}">')
        out.append(f'    <parent link="{parent}"/><child link="{child}"/>')
        out.append(f'    <origin xyz="{_fmt(xyz)}" rpy="{_fmt(rpy)}"/>')
        if axis is not None:
            out.append(f'    <axis xyz="{_AXES[axis]}"/>')
        if limits is not None:
            out.append(f'    <limit lower="{limits[0]!r}" upper="{limits[1]!r}"/>')
        out.append("  </joint>")
    out.append("</robot>")
    return "\n".join(out) + "\n"


def _spheres_yaml(spheres: dict) -> str:
    out = []
    for link, group in spheres.items():
        out.append(f"{link}:")
        for x, y, z, r in group:
            out.append(f"  - {{x: {float(x)!r}, y: {float(y)!r}, z: {float(z)!r}, r: {float(r)!r}}}")
    return "\n".join(out) + "\n"


def _prefixed_arm(prefix: str, mount_parent: str, xyz, rpy):
    links = tuple(prefix + ln for ln in _ARM7_LINKS)
    joints = [(f"{prefix}mount", "fixed", mount_parent, prefix + "base_link", xyz, None, None, rpy)]
    for jn, kind, parent, child, jxyz, axis, lim in _ARM7_JOINTS:
        joints.append((prefix + jn, kind, prefix + parent, prefix + child, jxyz, axis, lim))
    spheres = {prefix + ln: group for ln, group in _ARM7_SPHERES.items()}
    return links, joints, spheres


def _fetch_standin():
    links = ["mobile_base", "torso"]
    joints = [("torso_lift", "prismatic", "mobile_base", "torso", (0, 0, 0.35), "z", (0.0, 0.4))]
    spheres = {"mobile_base": [(0, 0, 0.15, 0.3)],
               "torso": [(0, 0, 0.1, 0.15), (0, 0, 0.25, 0.15)]}
    arm_links, arm_joints, arm_spheres = _prefixed_arm("", "torso", (0.1, 0, 0.3), (0, 0, 0))
    return (tuple(links) + arm_links, tuple(joints + arm_joints), {**spheres, **arm_spheres})


def _baxter_standin():
    links = ["pedestal", "torso"]
    joints = [("torso_mount", "fixed", "pedestal", "torso", (0, 0, 0.6), None, None)]
    spheres = {"pedestal": [(0, 0, 0.3, 0.25)],
               "torso": [(0, 0, 0.05, 0.15), (0, 0, 0.3, 0.15)]}
    all_links = list(links)
    all_joints = list(joints)
    for prefix, side in (("left_", 1.0), ("right_", -1.0)):
        arm_links, arm_joints, arm_spheres = _prefixed_arm(
            prefix, "torso", (0.05, 0.25 * side, 0.3), (0, 0, 0.785 * side))
        all_links += arm_links
        all_joints += arm_joints
        spheres.update(arm_spheres)
    return tuple(all_links), tuple(all_joints), spheres


def robot_texts(name: str) -> tuple[str, str]:
    """(URDF, sphere-model YAML) for a known robot name."""
    if name == "arm7":
        links, joints, spheres = _ARM7_LINKS, _ARM7_JOINTS, _ARM7_SPHERES
    elif name == "planar2":
        links, joints, spheres = _PLANAR2_LINKS, _PLANAR2_JOINTS, _PLANAR2_SPHERES
    elif name == "fetch_standin":
        links, joints, spheres = _fetch_standin()
    elif name == "baxter_standin":
        links, joints, spheres = _baxter_standin()
    else:
        raise KeyError(f"unknown robot {name!r}; known: {ROBOTS}")
    return _urdf(name, links, joints), _spheres_yaml(spheres)


ROBOTS = ("arm7", "planar2", "fetch_standin", "baxter_standin")
#: BASELINE.json model name -> synthetic stand-in actually used
STANDIN_FOR = {"panda": "arm7", "fetch": "fetch_standin", "baxter": "baxter_standin"}


@dataclass(frozen=True)
class Robot:
    """Compiled robot bundle (mirror of reference planners.py:48-56)."""

    tree: KinematicTree
    model: SphereModel
    pairs: SelfCollisionPairs
    program: KinematicProgram
    limits: np.ndarray
    name: str = "robot"


def build_robot(tree: KinematicTree, model: SphereModel, ignore_pairs=None,
                name: str = "robot") -> Robot:
    """trace -> optimize -> schedule, plus default self pairs (reference planners.py:59-68)."""
    pairs = default_self_collision_pairs(tree, ignore_pairs)
    program = schedule_program(optimize_graph(trace_kinematics(tree, model)))
    return Robot(tree=tree, model=model, pairs=pairs, program=program,
                 limits=tree.joint_limits(), name=name)


def load_robot(name: str) -> Robot:
    """Compiled bundle of a known robot; BASELINE names map to their stand-ins."""
    return _load(STANDIN_FOR.get(name, name))


@lru_cache(maxsize=None)
def _load(name: str) -> Robot:
    urdf, spheres = robot_texts(name)
    tree = parse_urdf(urdf)
    return build_robot(tree, load_sphere_model(tree, spheres), name=name)
