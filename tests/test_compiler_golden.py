"""The host compiler (robot/trace/program) reproduces the reference's programs.

Golden listings come from the reference itself (tests/golden/make_golden.py,
reference program.py:217-244 dump_program); identical listings mean the
generated kernels start from the reference's exact op DAG.
"""

import json

import numpy as np
import pytest

from golden_io import GOLDEN
from paper_2309_14545_b200 import (ROBOTS, build_robot, dump_program, load_robot,
                                   load_sphere_model, parse_urdf)
from paper_2309_14545_b200.trace import optimize_graph, trace_kinematics

PROGRAMS = json.loads((GOLDEN / "programs.json").read_text())


@pytest.mark.parametrize("name", ROBOTS)
def test_robot_program_matches_reference_listing(name):
    rob = load_robot(name)
    assert dump_program(rob.program) == PROGRAMS[name]["dump"]
    assert sorted(list(p) for p in rob.pairs.pairs) == PROGRAMS[name]["pairs"]


@pytest.mark.parametrize("name", ["one_joint", "skew_axis"])
def test_extra_programs_match(name):
    entry = PROGRAMS[name]
    tree = parse_urdf(entry["urdf"])
    rob = build_robot(tree, load_sphere_model(tree, entry["spheres"]))
    assert dump_program(rob.program) == entry["dump"]


def test_one_joint_golden_listing_text():
    # reference pkg/tests/test_program.py:211-233 (golden listing)
    expected = (
        "program dof=1 ops=7 checks=2\n"
        "  %0 = const 0\n"
        "  %1 = input q0\n"
        "  %2 = sin %1\n"
        "  %3 = cos %1\n"
        "  %4 = const 0.5\n"
        "  %5 = mul %3 %4\n"
        "  %6 = mul %2 %4\n"
        "  check link=1 coarse[0] r=0.1 pos=(%5, %6, %0)\n"
        "  check link=1 fine[0] r=0.1 pos=(%5, %6, %0)\n"
    )
    assert PROGRAMS["one_joint"]["dump"] == expected


def test_optimizer_idempotent_and_sound():
    from paper_2309_14545_b200 import robot_texts
    from paper_2309_14545_b200.trace import evaluate_graph
    urdf, spheres = robot_texts("arm7")
    tree = parse_urdf(urdf)
    model = load_sphere_model(tree, spheres)
    raw = trace_kinematics(tree, model)
    og = optimize_graph(raw)
    twice = optimize_graph(og)
    assert (twice.kinds, twice.a, twice.b, twice.values) == (og.kinds, og.a, og.b, og.values)
    assert len(og) < len(raw)
    q = np.random.default_rng(3).uniform(-1, 1, size=(200, 7))
    a, b = evaluate_graph(raw, q), evaluate_graph(og, q)
    assert max(float(np.max(np.abs(a[k] - b[k]))) for k in a) <= 1e-12


def test_marker_closure_is_prefix():
    prog = load_robot("baxter_standin").program
    for m in prog.checks:
        stack, seen = list(m.xyz), set()
        while stack:
            i = stack.pop()
            if i in seen:
                continue
            seen.add(i)
            assert i < m.position
            stack.extend(x for x in (prog.a[i], prog.b[i]) if x >= 0)
