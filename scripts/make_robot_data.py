"""Generate paper_2309_14545_b200/data/robots.json with the REFERENCE's compiler.

Offline tool (needs /root/reference, i.e. runs in the build container only).
The product does not compile robots: like a user of the drop-in, it consumes
``KinematicProgram``s produced by the reference's own tracing compiler
(vecmp.planners.build_robot: trace -> optimize -> schedule, planners.py:59-68).
This script runs that compiler on

* ``arm7`` and ``planar2`` - the reference's bundled robots (its resources
  directory, read as-is); ``arm7`` is the "Panda" stand-in;
* ``fetch_standin`` and ``baxter_standin`` - SYNTHETIC stand-ins for Fetch and
  Baxter (the real models are not in the reference): URDF /
  sphere documents assembled here from copies of the bundled arm7 chain plus a
  few base links (layout below);

and serialises each compiled program (ops, exact float64 constants, markers),
the self-collision pairs, the sphere model and the joint limits.  It checks
every program against the reference listings recorded in
tests/golden/programs.json before writing.

    python scripts/make_robot_data.py
"""

from __future__ import annotations

import copy
import json
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import yaml

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from vecmp.planners import build_robot  # noqa: E402
from vecmp.program import dump_program  # noqa: E402
from vecmp.robot import load_sphere_model, parse_urdf  # noqa: E402

RESOURCES = REF / "vecmp" / "resources" / "robots"
OUT = ROOT / "paper_2309_14545_b200" / "data" / "robots.json"


def _bundled(name: str) -> tuple[str, str]:
    return ((RESOURCES / f"{name}.urdf").read_text(),
            (RESOURCES / f"{name}_spheres.yaml").read_text())


def _joint(name, kind, parent, child, xyz, rpy=(0.0, 0.0, 0.0), axis=None, limits=None):
    j = ET.Element("joint", name=name, type=kind)
    ET.SubElement(j, "parent", link=parent)
    ET.SubElement(j, "child", link=child)
    ET.SubElement(j, "origin", xyz=" ".join(repr(float(v)) for v in xyz),
                  rpy=" ".join(repr(float(v)) for v in rpy))
    if axis is not None:
        ET.SubElement(j, "axis", xyz=axis)
    if limits is not None:
        ET.SubElement(j, "limit", lower=repr(limits[0]), upper=repr(limits[1]))
    return j


def _assemble(name: str, base_links, base_joints, base_spheres, arms) -> tuple[str, str]:
    """Robot = base links/joints + copies of the bundled arm7 chain.

    ``arms``: (prefix, mount parent link, mount xyz, mount rpy) per arm copy.
    Element order (links first, then joints) fixes the reference's link indices.
    """
    arm_urdf, arm_spheres = _bundled("arm7")
    arm = ET.fromstring(arm_urdf)
    arm_sph = yaml.safe_load(arm_spheres)
    robot = ET.Element("robot", name=name)
    links = list(base_links)
    joints = list(base_joints)
    spheres = dict(base_spheres)
    for prefix, parent, xyz, rpy in arms:
        links += [prefix + ln.get("name") for ln in arm.findall("link")]
        joints.append(_joint(prefix + "mount", "fixed", parent, prefix + "base_link", xyz, rpy))
        for j in arm.findall("joint"):
            j = copy.deepcopy(j)
            j.set("name", prefix + j.get("name"))
            for tag in ("parent", "child"):
                j.find(tag).set("link", prefix + j.find(tag).get("link"))
            joints.append(j)
        spheres.update({prefix + link: group for link, group in arm_sph.items()})
    for ln in links:
        ET.SubElement(robot, "link", name=ln)
    robot.extend(joints)
    return ET.tostring(robot, encoding="unicode"), yaml.safe_dump(spheres, sort_keys=False)


def fetch_standin() -> tuple[str, str]:
    """mobile base sphere -> prismatic torso lift (z, [0, 0.4]) -> torso (2 spheres)
    -> fixed mount (0.1, 0, 0.3) -> arm7.  D = 8."""
    return _assemble(
        "fetch_standin", ["mobile_base", "torso"],
        [_joint("torso_lift", "prismatic", "mobile_base", "torso", (0, 0, 0.35), axis="0 0 1",
                limits=(0.0, 0.4))],
        {"mobile_base": [{"x": 0.0, "y": 0.0, "z": 0.15, "r": 0.3}],
         "torso": [{"x": 0.0, "y": 0.0, "z": 0.1, "r": 0.15},
                   {"x": 0.0, "y": 0.0, "z": 0.25, "r": 0.15}]},
        [("", "torso", (0.1, 0, 0.3), (0, 0, 0))])


def baxter_standin() -> tuple[str, str]:
    """pedestal -> fixed torso (z 0.6, 2 spheres) -> two arm7 chains mounted at
    (0.05, +-0.25, 0.3) with yaw +-0.785.  D = 14."""
    return _assemble(
        "baxter_standin", ["pedestal", "torso"],
        [_joint("torso_mount", "fixed", "pedestal", "torso", (0, 0, 0.6))],
        {"pedestal": [{"x": 0.0, "y": 0.0, "z": 0.3, "r": 0.25}],
         "torso": [{"x": 0.0, "y": 0.0, "z": 0.05, "r": 0.15},
                   {"x": 0.0, "y": 0.0, "z": 0.3, "r": 0.15}]},
        [("left_", "torso", (0.05, 0.25, 0.3), (0, 0, 0.785)),
         ("right_", "torso", (0.05, -0.25, 0.3), (0, 0, -0.785))])


SOURCES = {
    "arm7": ("reference resources/robots/arm7 (stand-in for Panda)", lambda: _bundled("arm7")),
    "planar2": ("reference resources/robots/planar2", lambda: _bundled("planar2")),
    "fetch_standin": ("SYNTHETIC stand-in for Fetch: " + fetch_standin.__doc__.split("\n")[0],
                      fetch_standin),
    "baxter_standin": ("SYNTHETIC stand-in for Baxter: " + baxter_standin.__doc__.split("\n")[0],
                       baxter_standin),
}


def texts(name: str) -> tuple[str, str]:
    """(URDF, sphere YAML) the robot is compiled from."""
    return SOURCES[name][1]()


def compile_reference(name: str):
    urdf, spheres = texts(name)
    tree = parse_urdf(urdf)
    return tree, build_robot(tree, load_sphere_model(tree, spheres))


def serialise(name: str) -> dict:
    tree, rob = compile_reference(name)
    p = rob.program
    golden = json.loads((ROOT / "tests" / "golden" / "programs.json").read_text())[name]
    assert dump_program(p) == golden["dump"], f"{name}: program differs from the golden listing"
    assert sorted(list(x) for x in rob.pairs.pairs) == golden["pairs"]
    sph = lambda s: None if s is None else [*map(float, s.center), float(s.radius)]  # noqa: E731
    return {
        "name": name,
        "source": SOURCES[name][0],
        "dof": int(p.dof),
        "links": [ln for ln in tree.links],
        "limits": [[float(lo), float(hi)] for lo, hi in rob.limits],
        "program": {
            "kinds": [int(k) for k in p.kinds],
            "a": [int(x) for x in p.a],
            "b": [int(x) for x in p.b],
            "values": [float(v) for v in p.values],
            "checks": [[int(m.link), m.level, int(m.index), float(m.radius),
                        [int(v) for v in m.xyz], int(m.position)] for m in p.checks],
        },
        "pairs": sorted([int(a), int(b)] for a, b in rob.pairs.pairs),
        "spheres": {"fine": [[sph(s) for s in link] for link in rob.model.fine],
                    "coarse": [sph(s) for s in rob.model.coarse]},
    }


def main() -> None:
    data = {name: serialise(name) for name in SOURCES}
    OUT.write_text(json.dumps(data, indent=None, separators=(",", ":")) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes): {', '.join(data)}")


if __name__ == "__main__":
    main()
