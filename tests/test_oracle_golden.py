"""Pin the CPU oracle (oracle/vecmp_oracle.py) to outputs of the reference itself.

Every fixture was produced by running the reference package (make_golden.py);
the oracle must reproduce float32 results bit for bit and verdicts exactly.
Only once this passes is the oracle trusted as the GPU parity checker.
"""

import numpy as np
import pytest

import golden_io
import vecmp_oracle as O
from paper_2309_14545_b200 import load_robot

ROBOTS = ("planar2", "arm7", "fetch_standin", "baxter_standin")
FK = golden_io.load("fk")
BLOCKS = golden_io.load("blocks")
MOTION = golden_io.load("motion")
LANES = golden_io.load("lanes")
NARROW = golden_io.load("narrow")


@pytest.mark.parametrize("name", ROBOTS)
def test_f32_interpreter_bitwise(name):
    prog = load_robot(name).program
    rows = O.rows_f32(prog, FK[f"q_{name}"])
    assert np.array_equal(O.marker_centres(prog, rows), FK[f"f32_{name}"])


@pytest.mark.parametrize("name", ROBOTS)
def test_f64_fk_matches_evaluate_graph_and_chain(name):
    prog = load_robot(name).program
    cen = O.marker_centres(prog, O.rows_f64(prog, FK[f"q_{name}"]))
    assert np.allclose(cen, FK[f"f64_{name}"], rtol=0, atol=1e-12)
    chain = FK[f"chain_{name}"]                         # (16, markers, 3) 4x4 chain oracle
    assert np.max(np.abs(cen[:, :, :16].transpose(2, 0, 1) - chain)) < 1e-9


def _block_cases():
    for name in ROBOTS:
        e = 0
        while f"env_{name}_{e}_kinds" in BLOCKS:
            yield name, e
            e += 1


@pytest.mark.parametrize("name,e", list(_block_cases()))
def test_block_verdicts(name, e):
    rob = load_robot(name)
    env = golden_io.env_from(BLOCKS, f"env_{name}_{e}")
    ob = O.Obstacles(env.primitives)
    q = BLOCKS[f"q_{name}"]
    n = q.shape[1]
    for prune in (1, 0):
        got = np.concatenate([O.validate_lanes(rob.program, rob.pairs, ob, q[:, i:i + 8],
                                               prune=bool(prune)) for i in range(0, n, 8)])
        assert np.array_equal(got, BLOCKS[f"v_{name}_{e}_w8_p{prune}"])
    wide = O.validate_lanes(rob.program, rob.pairs, ob, q, prune=True)
    assert np.array_equal(wide, BLOCKS[f"v_{name}_{e}_wide"])
    strict = np.concatenate([O.validate_lanes(rob.program, rob.pairs, ob, q[:, i:i + 8],
                                              reject_all=True) for i in range(0, n, 8)])
    assert np.array_equal(strict, BLOCKS[f"v_{name}_{e}_reject_all"])


def _motion_keys():
    return sorted({k[len("starts_"):] for k in MOTION.files if k.startswith("starts_")})


@pytest.mark.parametrize("key", _motion_keys())
def test_rake_verdicts_and_block_counts(key):
    robot = key.rsplit("_", 1)[0]
    rob = load_robot(robot)
    env = golden_io.env_from(MOTION, f"env_{key}")
    ob = O.Obstacles(env.primitives)
    s, g, res = MOTION[f"starts_{key}"], MOTION[f"goals_{key}"], float(MOTION[f"res_{key}"])
    assert [O.discretization(a, b, res) for a, b in zip(s, g)] == MOTION[f"n_{key}"].tolist()
    dense = [O.edge_all_states(rob.program, rob.pairs, ob, a, b, res)[1] for a, b in zip(s, g)]
    for width in (8, 1, 32):
        for bwd in (0, 1):
            tag = f"{key}_w{width}_b{bwd}"
            implied = [O.rake_blocks_from_states(v, width, bool(bwd)) for v in dense]
            assert [v for v, _ in implied] == MOTION[f"verdict_{tag}"].tolist()
            assert [b for _, b in implied] == MOTION[f"blocks_{tag}"].tolist()
    # the block-by-block restatement agrees too (W = 8, forward), on a subset
    for i in range(0, len(s), 7):
        assert O.rake_check(rob.program, rob.pairs, ob, s[i], g[i], res, 8) == (
            bool(MOTION[f"verdict_{key}_w8_b0"][i]), int(MOTION[f"blocks_{key}_w8_b0"][i]))


@pytest.mark.parametrize("d", range(1, 17))
def test_l2_and_discretization_bitwise(d):
    a, b = LANES[f"a_{d}"], LANES[f"b_{d}"]
    assert [O.np_l2(x, y) for x, y in zip(a, b)] == LANES[f"l2_{d}"].tolist()
    for tag, res in (("r32", 1.0 / 32.0), ("r05", 0.05), ("r07", 0.07)):
        assert [O.discretization(x, y, res) for x, y in zip(a, b)] == LANES[f"n_{tag}_{d}"].tolist()


def test_narrowphase_cases():
    from paper_2309_14545_b200.collision import BoxObstacle, CapsuleObstacle, SphereObstacle
    N = NARROW
    for i in range(len(N["sph_r"])):
        ob = O.Obstacles([SphereObstacle(center=N["sph_c"][i], radius=float(N["sph_r"][i]))])
        h = O.kind_hits(ob, N["sph_pts"][i].T.copy(), float(N["sph_rs"][i]))[0][0]
        assert np.array_equal(h, N["sph_hits"][i])
    for i in range(len(N["cap_r"])):
        ob = O.Obstacles([CapsuleObstacle(p0=N["cap_p0"][i], p1=N["cap_p1"][i],
                                          radius=float(N["cap_r"][i]))])
        h = O.kind_hits(ob, N["cap_pts"][i].T.copy(), float(N["cap_rs"][i]))[1][0]
        assert np.array_equal(h, N["cap_hits"][i])
    for i in range(len(N["box_rs"])):
        ob = O.Obstacles([BoxObstacle(center=N["box_c"][i], half_extents=N["box_h"][i],
                                      rotation=N["box_rot"][i])])
        h = O.kind_hits(ob, N["box_pts"][i].T.copy(), float(N["box_rs"][i]))[2][0]
        assert np.array_equal(h, N["box_hits"][i])


def test_reference_float32_verdicts_agree_with_f64_sign_outside_band():
    """The reference's own verdicts equal sign(clearance) away from the 1e-4 m band."""
    rob = load_robot("arm7")
    for e in range(3):
        env = golden_io.env_from(BLOCKS, f"env_arm7_{e}")
        q = BLOCKS["q_arm7"]
        c = O.clearance_f64(rob.program, rob.pairs, env.primitives, q)
        outside = np.abs(c) > 1e-4
        assert np.array_equal(BLOCKS[f"v_arm7_{e}_wide"][outside], (c > 0)[outside])
