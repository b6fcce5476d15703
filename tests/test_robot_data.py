"""The bundled robot programs are the reference compiler's programs.

``paper_2309_14545_b200/data/robots.json`` is written by
scripts/make_robot_data.py with the reference's own tracing compiler; these
tests pin the shipped data against the reference's program listings recorded
independently by tests/golden/make_golden.py (reference program.py:217-244
``dump_program`` format), so the kernels start from the reference's exact op
DAG, self pairs and limits.
"""

import json

import numpy as np
import pytest

from golden_io import GOLDEN
from paper_2309_14545_b200 import ROBOTS, load_robot
from paper_2309_14545_b200.program import CONST, INPUT, NEG, SIN, COS

PROGRAMS = json.loads((GOLDEN / "programs.json").read_text())
NAMES = {2: "add", 3: "sub", 4: "mul", 5: "neg", 6: "sin", 7: "cos"}


def listing(program) -> str:
    """The reference's listing format (program.py:217-244), restated for the check."""
    out = [f"program dof={program.dof} ops={len(program)} checks={len(program.checks)}"]
    at: dict = {}
    for m in program.checks:
        at.setdefault(m.position, []).append(m)

    def markers(pos):
        for m in at.get(pos, ()):
            x, y, z = m.xyz
            out.append(f"  check link={m.link} {m.level}[{m.index}] r={m.radius:.6g} "
                       f"pos=(%{x}, %{y}, %{z})")
    for i, k in enumerate(int(k) for k in program.kinds):
        markers(i)
        if k == CONST:
            body = f"const {program.values[i]:.9g}"
        elif k == INPUT:
            body = f"input q{int(program.values[i])}"
        elif k in (NEG, SIN, COS):
            body = f"{NAMES[k]} %{program.a[i]}"
        else:
            body = f"{NAMES[k]} %{program.a[i]} %{program.b[i]}"
        out.append(f"  %{i} = {body}")
    markers(len(program))
    return "\n".join(out) + "\n"


@pytest.mark.parametrize("name", ROBOTS)
def test_program_matches_reference_listing(name):
    rob = load_robot(name)
    assert listing(rob.program) == PROGRAMS[name]["dump"]
    assert sorted(list(p) for p in rob.pairs.pairs) == PROGRAMS[name]["pairs"]


@pytest.mark.parametrize("name", ROBOTS)
def test_robot_bundle_shapes(name):
    rob = load_robot(name)
    p = rob.program
    assert rob.limits.shape == (p.dof, 2) and (rob.limits[:, 0] < rob.limits[:, 1]).all()
    assert p.kinds.dtype == np.int8 and p.values.dtype == np.float64
    assert len(p.kinds) == len(p.a) == len(p.b) == len(p.values)
    # every marker reads ops that precede it; fine markers carry model radii
    for m in p.checks:
        assert max(m.xyz) < m.position <= len(p)
    fine = [m for m in p.checks if m.level == "fine"]
    assert [m.radius for m in fine] == [s[3] for link in rob.model.fine for s in link]
    assert set(rob.model.checked_links()) == {m.link for m in fine}


def test_standin_names():
    assert load_robot("panda") is load_robot("arm7")
    assert load_robot("fetch").program.dof == 8 and load_robot("baxter").program.dof == 14
    with pytest.raises(KeyError):
        load_robot("ur5")
