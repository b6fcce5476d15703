"""GPU parity: the sm_100a kernels (through the C ABI / reference-signature
shims) against the pinned oracle and the reference's own golden outputs.

Bars (BASELINE.json north_star):
  * sphere centres within 1e-5 m of the float64 values;
  * collision verdicts bit-identical for every configuration whose |minimum
    signed clearance| > 1e-4 m; mismatches inside the band are counted;
  * motion verdicts identical under the same resolution rule (and the
    reference's rake block counts reproduced for the context width).
"""

import numpy as np
import pytest

import golden_io
import vecmp_oracle as O
from paper_2309_14545_b200 import (ConfigBlock, Scratch, ValidationContext, evaluate_program,
                                   load_robot, soa_from_aos, validate_block, workloads)
from paper_2309_14545_b200 import motion as M
from paper_2309_14545_b200 import runtime

pytestmark = pytest.mark.gpu

ROBOTS = ("planar2", "arm7", "fetch_standin", "baxter_standin")
BAND = 1e-4
CENTRE_TOL = 1e-5


def _verdict_parity(rob, prims, q, got):
    """Assert bit-identical verdicts outside the band; return in-band mismatch count."""
    ref = O.validate_configs(rob.program, rob.pairs, prims, q)
    clear = O.clearance_f64(rob.program, rob.pairs, prims, q)
    outside = np.abs(clear) > BAND
    bad = np.flatnonzero(outside & (got != ref))
    assert bad.size == 0, f"{bad.size} verdicts differ outside the band, e.g. {bad[:5]}"
    return int(np.sum(~outside & (got != ref)))


# ------------------------------------------------------------------ FK

@pytest.mark.parametrize("name", ROBOTS)
def test_fk_centres_within_1e5_of_float64(cuda, name):
    fk = golden_io.load("fk")
    rob = load_robot(name)
    q = fk[f"q_{name}"]
    cen = runtime.fk_spheres(rob.program, q).cpu().numpy().reshape(-1, 3, q.shape[1])
    assert np.max(np.abs(cen - fk[f"f64_{name}"])) <= CENTRE_TOL
    # and close to the reference's own float32 stream
    assert np.max(np.abs(cen - fk[f"f32_{name}"])) <= CENTRE_TOL


@pytest.mark.parametrize("name", ROBOTS)
def test_fk_large_batch_vs_float64(cuda, name):
    rob = load_robot(name)
    q = workloads.uniform_configs(rob.limits, 100_000, 7)
    cen = runtime.fk_spheres(rob.program, q).cpu().numpy().reshape(-1, 3, q.shape[1])
    ref = O.marker_centres(rob.program, O.rows_f64(rob.program, q))
    assert np.max(np.abs(cen - ref)) <= CENTRE_TOL


def test_evaluate_program_sink_and_rows(cuda):
    rob = load_robot("arm7")
    rng = np.random.default_rng(31)
    configs = [rng.uniform(rob.limits[:, 0], rob.limits[:, 1]).astype(np.float32) for _ in range(8)]

    class Rec:
        def __init__(self, stop=None):
            self.calls, self.stop = [], stop

        def __call__(self, m, x, y, z):
            self.calls.append((m, x.copy(), y.copy(), z.copy()))
            return self.stop is not None and len(self.calls) >= self.stop

    wide = Rec()
    scratch = evaluate_program(rob.program, soa_from_aos(configs, width=8), wide)
    assert isinstance(scratch, Scratch) and scratch.rows.shape == (len(rob.program), 8)
    assert len(wide.calls) == len(rob.program.checks)
    for k, q in enumerate(configs):            # lanes == width-1 runs, bitwise
        narrow = Rec()
        evaluate_program(rob.program, soa_from_aos([q], width=1), narrow)
        for (mw, xw, yw, zw), (mn, xn, yn, zn) in zip(wide.calls, narrow.calls):
            assert mw is mn and xw[k] == xn[0] and yw[k] == yn[0] and zw[k] == zn[0]
    partial = Rec(stop=3)
    evaluate_program(rob.program, soa_from_aos(configs, width=8), partial)
    assert len(partial.calls) == 3
    with pytest.raises(ValueError):
        evaluate_program(rob.program, soa_from_aos([np.zeros(3, np.float32)]), None)


# ------------------------------------------------------------- blocks

def _block_cases():
    fx = golden_io.load("blocks")
    for name in ROBOTS:
        e = 0
        while f"env_{name}_{e}_kinds" in fx:
            yield name, e
            e += 1


@pytest.mark.parametrize("name,e", list(_block_cases()))
def test_validate_block_vs_reference_goldens(cuda, name, e):
    fx = golden_io.load("blocks")
    rob = load_robot(name)
    env = golden_io.env_from(fx, f"env_{name}_{e}")
    q = fx[f"q_{name}"]
    n = q.shape[1]
    clear = O.clearance_f64(rob.program, rob.pairs, env.primitives, q)
    outside = np.abs(clear) > BAND
    for prune in (True, False):
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, env, width=8, prune=prune)
        got = np.concatenate([ctx.validate_block(ConfigBlock(rob.program.dof, 8,
                                                             np.ascontiguousarray(q[:, i:i + 8]), 8))
                              for i in range(0, n, 8)])
        ref = fx[f"v_{name}_{e}_w8_p{int(prune)}"]
        assert np.array_equal(got[outside], ref[outside])
        assert ctx.blocks_evaluated == n // 8
    wide = validate_block(rob.program, rob.model, rob.pairs, env,
                          ConfigBlock(rob.program.dof, n, q, n))
    assert np.array_equal(wide[outside], fx[f"v_{name}_{e}_wide"][outside])
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, env, width=8)
    strict = np.concatenate([ctx.validate_block(ConfigBlock(rob.program.dof, 8,
                                                            np.ascontiguousarray(q[:, i:i + 8]), 8),
                                                reject_all=True) for i in range(0, n, 8)])
    blk_out = outside.reshape(-1, 8).all(axis=1).repeat(8)
    assert np.array_equal(strict[blk_out], fx[f"v_{name}_{e}_reject_all"][blk_out])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg3", "cfg4", "cfg5_16", "cfg5_128", "cfg5_1024"])
def test_batch_workloads_vs_oracle(cuda, cfg):
    n = 65536 if cfg == "cfg1" else 16384
    wl = {"cfg1": lambda: workloads.config1(n), "cfg3": lambda: workloads.config3(n),
          "cfg4": lambda: workloads.config4(n)}.get(cfg, lambda: workloads.config5(n, int(cfg[5:])))()
    rob = load_robot(wl.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
    got = ctx.validate_configs(wl.q)
    band = _verdict_parity(rob, wl.env.primitives, wl.q, got)
    assert band <= max(2, n // 2000)
    rate = 1 - got.mean()
    assert 0.15 < rate < 0.65, f"collision rate {rate:.3f} outside the calibrated band"


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4"])
def test_full_size_batches_self_consistent(cuda, cfg):
    """1M-config batches: size-independent properties (the oracle checks a sample)."""
    torch = cuda
    wl = workloads.config3() if cfg == "cfg3" else workloads.config4()
    rob = load_robot(wl.robot)
    n = wl.q.shape[1]
    qd = torch.from_numpy(wl.q).cuda()
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
    early = ctx.validate_batch(qd).cpu().numpy()
    dense = ctx.validate_batch(qd, early_exit=False).cpu().numpy()
    assert np.array_equal(early, dense)                      # early exit never changes verdicts
    noprune = ValidationContext(rob.program, rob.model, rob.pairs, wl.env, prune=False)
    assert np.array_equal(noprune.validate_batch(qd).cpu().numpy(), early)   # prune is sound
    # chunked launches with a leading dimension == one launch
    half = n // 2 + 17
    a = runtime.unpack_bits(ctx.validate_batch(qd[:, :half]).cpu().numpy(), half)
    b = runtime.unpack_bits(ctx.validate_batch(qd[:, half:]).cpu().numpy(), n - half)
    full = runtime.unpack_bits(early, n)
    assert np.array_equal(np.concatenate([a, b]), full)
    idx = np.random.default_rng(5).choice(n, 8192, replace=False)
    _verdict_parity(rob, wl.env.primitives, wl.q[:, idx], full[idx])


def test_padding_permutation_and_edges(cuda):
    rob = load_robot("arm7")
    env = workloads.config2_scene()
    rng = np.random.default_rng(61)
    configs = [rng.uniform(rob.limits[:, 0], rob.limits[:, 1]).astype(np.float32) for _ in range(8)]
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, env)
    base = ctx.validate_block(soa_from_aos(configs, width=8))
    perm = rng.permutation(8)
    assert np.array_equal(ctx.validate_block(soa_from_aos([configs[p] for p in perm])), base[perm])
    one = ctx.validate_block(soa_from_aos(configs[:3], width=8))[:3]
    assert np.array_equal(one, base[:3])
    assert ctx.state_valid(configs[0]) == bool(base[0])
    from paper_2309_14545_b200 import Environment, SphereObstacle
    empty = ValidationContext(rob.program, rob.model, rob.pairs, Environment())
    assert empty.validate_configs(np.zeros((7, 5), np.float32)).all()
    engulf = ValidationContext(rob.program, rob.model, rob.pairs,
                               Environment([SphereObstacle(np.zeros(3), 5.0)]))
    assert not engulf.validate_configs(np.zeros((7, 100), np.float32)).any()
    assert engulf.validate_configs(np.zeros((7, 0), np.float32)).size == 0


def test_block_validator_sink_matches_fused_path(cuda):
    """The GPU-backed BlockValidator sink (reference collision.py:293-408) driven
    by evaluate_program gives the fused kernel's verdicts, and aborts early."""
    from paper_2309_14545_b200 import BlockValidator, Environment, SphereObstacle
    fx = golden_io.load("blocks")
    rob = load_robot("arm7")
    env = golden_io.env_from(fx, "env_arm7_4")
    q = fx["q_arm7"][:, :64]
    fused = validate_block(rob.program, rob.model, rob.pairs, env, ConfigBlock(7, 64, q, 64))
    for reject_all in (False, True):
        sink = BlockValidator(env.packed(), rob.pairs, width=64, reject_all=reject_all)
        evaluate_program(rob.program, ConfigBlock(7, 64, np.ascontiguousarray(q), 64), sink)
        expect = np.zeros(64, bool) if reject_all and not fused.all() else fused
        assert np.array_equal(sink.result(), expect)
    engulf = Environment([SphereObstacle(np.zeros(3), 3.0)])
    calls = []

    def counting(m, x, y, z, inner=BlockValidator(engulf.packed(), rob.pairs, width=8)):
        calls.append(m)
        counting.inner = inner
        return inner(m, x, y, z)

    evaluate_program(rob.program, soa_from_aos([q[:, 0].copy()], width=8), counting)
    assert not counting.inner.result().any()
    assert len(calls) < len(rob.program.checks)


def test_validate_block_drives_caller_sink(cuda):
    """validate_block(..., sink=s) resets s, drives it through evaluate_program
    and returns s.result() (reference collision.py:422-429)."""
    from paper_2309_14545_b200 import BlockValidator
    fx = golden_io.load("blocks")
    rob = load_robot("arm7")
    env = golden_io.env_from(fx, "env_arm7_4")
    q = np.ascontiguousarray(fx["q_arm7"][:, :64])
    outside = np.abs(O.clearance_f64(rob.program, rob.pairs, env.primitives, q)) > BAND
    for reject_all in (False, True):
        ref = fx[f"v_arm7_4_{'reject_all' if reject_all else 'w8_p1'}"][:64]
        sink = BlockValidator(env.packed(), rob.pairs, width=8, reject_all=not reject_all)
        sink.valid[:] = False                      # stale state: validate_block resets it
        got = []
        for i in range(0, 64, 8):
            out = validate_block(rob.program, rob.model, rob.pairs, env,
                                 ConfigBlock(7, 8, np.ascontiguousarray(q[:, i:i + 8]), 8),
                                 reject_all=reject_all, sink=sink)
            assert np.array_equal(out, sink.result()) and sink.reject_all == reject_all
            got.append(out)
        got = np.concatenate(got)
        blk = outside.reshape(-1, 8).all(axis=1).repeat(8) if reject_all else outside
        assert np.array_equal(got[blk], ref[blk])

    class Recorder:                                # any object with the sink protocol
        def __init__(self):
            self.resets, self.calls = [], 0

        def reset(self, prune=None, reject_all=None):
            self.resets.append((prune, reject_all))

        def __call__(self, marker, x, y, z):
            self.calls += 1
            return False

        def result(self):
            return np.full(8, True)

    rec = Recorder()
    out = validate_block(rob.program, rob.model, rob.pairs, env,
                         ConfigBlock(7, 8, np.ascontiguousarray(q[:, :8]), 8), prune=False,
                         sink=rec)
    assert out.all() and rec.resets == [(False, False)] and rec.calls == len(rob.program.checks)


@pytest.mark.parametrize("width,backward", [(32, False), (32, True), (8, False), (8, True),
                                            (5, True), (1, False)])
def test_rake_states_bit_exact(cuda, width, backward):
    """Every state the rake visits (vmp_motion_states: the rake kernels' index
    math, vmp_rake_param and vmp_lerp_exact) equals the reference's
    interpolate_lanes at t = f32(i / n) bit for bit, in the reference's
    stratum order (motion.py:32-78, lanes.py:91-103)."""
    mw = workloads.config2()
    E = 512
    s, g = mw.starts[:E], mw.goals[:E]
    n, off, idx, st = runtime.motion_states(runtime.to_device(s), runtime.to_device(g),
                                            mw.resolution, width=width, backward=backward)
    for e in range(E):
        ne = O.discretization(s[e], g[e], mw.resolution)
        assert n[e] == ne
        S = -(-ne // width)
        order = range(S, 0, -1) if backward else range(1, S + 1)
        exp = np.concatenate([np.arange(width, dtype=np.int64) * S + j for j in order])
        inr = exp <= ne
        got_idx = idx[off[e]:off[e + 1]]
        assert np.array_equal(got_idx, np.where(inr, exp, 0))
        ref = O.rake_states(s[e], g[e], ne, exp[inr]).T
        got = st[off[e]:off[e + 1]][inr]
        assert np.array_equal(got.view(np.uint32), np.ascontiguousarray(ref).view(np.uint32))


# ---------------------------------------------------------- narrowphase

def test_single_obstacle_lane_wrappers_vs_reference(cuda):
    from paper_2309_14545_b200 import (BoxObstacle, CapsuleObstacle, SphereObstacle,
                                       sphere_vs_capsule_lanes, sphere_vs_cuboid_lanes,
                                       sphere_vs_sphere_lanes)
    N = golden_io.load("narrow")
    mism = 0
    for i in range(0, len(N["sph_r"]), 3):
        h = sphere_vs_sphere_lanes(*N["sph_pts"][i].T, float(N["sph_rs"][i]),
                                   SphereObstacle(N["sph_c"][i], float(N["sph_r"][i])))
        mism += int(np.sum(h != N["sph_hits"][i]))
    for i in range(0, len(N["cap_r"]), 3):
        h = sphere_vs_capsule_lanes(*N["cap_pts"][i].T, float(N["cap_rs"][i]),
                                    CapsuleObstacle(N["cap_p0"][i], N["cap_p1"][i], float(N["cap_r"][i])))
        mism += int(np.sum(h != N["cap_hits"][i]))
    for i in list(range(50)) + list(range(50, len(N["box_rs"]), 3)):
        h = sphere_vs_cuboid_lanes(*N["box_pts"][i].T, float(N["box_rs"][i]),
                                   BoxObstacle(N["box_c"][i], N["box_h"][i], N["box_rot"][i]))
        mism += int(np.sum(h != N["box_hits"][i]))
    assert mism == 0


# --------------------------------------------------------------- motion

def _motion_keys():
    fx = golden_io.load("motion")
    return sorted({k[len("starts_"):] for k in fx.files if k.startswith("starts_")})


@pytest.mark.parametrize("key", _motion_keys())
def test_rake_vs_reference_goldens(cuda, key):
    fx = golden_io.load("motion")
    rob = load_robot(key.rsplit("_", 1)[0])
    env = golden_io.env_from(fx, f"env_{key}")
    s, g, res = fx[f"starts_{key}"], fx[f"goals_{key}"], float(fx[f"res_{key}"])
    ns = [M.discretization_count(a, b, res) for a, b in zip(s[:20], g[:20])]
    assert ns == fx[f"n_{key}"][:20].tolist()
    for width in (8, 1, 32):
        for bwd in (0, 1):
            tag = f"{key}_w{width}_b{bwd}"
            ctx = ValidationContext(rob.program, rob.model, rob.pairs, env, width=width)
            bits, n_states, blocks = M.validate_motions(ctx, s, g, res, backward=bool(bwd),
                                                        width=width, counts=True)
            verdict = runtime.unpack_bits(bits.cpu().numpy(), len(s))
            assert verdict.tolist() == fx[f"verdict_{tag}"].tolist()
            assert blocks.cpu().numpy().tolist() == fx[f"blocks_{tag}"].tolist()
            assert n_states.cpu().numpy().tolist() == fx[f"n_{key}"].tolist()
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, env, width=8)
    for i in range(0, len(s), 9):                       # the per-edge shim, too
        assert M.raked_motion_check(s[i], g[i], ctx, res) == (
            bool(fx[f"verdict_{key}_w8_b0"][i]), int(fx[f"blocks_{key}_w8_b0"][i]))


def test_cfg2_all_edges_vs_oracle(cuda):
    mw = workloads.config2()
    rob = load_robot("arm7")
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
    bits, n_states, blocks = M.validate_motions(ctx, mw.starts, mw.goals, mw.resolution, counts=True)
    verdict = runtime.unpack_bits(bits.cpu().numpy(), len(mw.starts))
    ob = O.Obstacles(mw.env.primitives)
    expect, ns = [], []
    for a, b in zip(mw.starts, mw.goals):
        n, v = O.edge_all_states(rob.program, rob.pairs, ob, a, b, mw.resolution)
        expect.append(bool(v.all()))
        ns.append(n)
    assert n_states.cpu().numpy().tolist() == ns
    assert verdict.tolist() == expect
    assert verdict[0::2].all()                         # forced-free edges
    assert 0.4 < verdict.mean() < 0.7


def test_discretize_bitwise_vs_reference(cuda):
    L = golden_io.load("lanes")
    for d in range(1, 17):
        a, b = L[f"a_{d}"], L[f"b_{d}"]
        for tag, res in (("r32", 1.0 / 32.0), ("r05", 0.05), ("r07", 0.07)):
            got = runtime.discretize_device(runtime.to_device(a), runtime.to_device(b), res)
            assert got.cpu().numpy().tolist() == L[f"n_{tag}_{d}"].tolist()


def test_motion_errors(cuda):
    rob = load_robot("planar2")
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, workloads.config2_scene())
    with pytest.raises(ValueError):
        M.raked_motion_check(np.zeros(2, np.float32), np.ones(2, np.float32), ctx, 0.0)
    with pytest.raises(ValueError):
        M.raked_motion_check(np.zeros(2, np.float32), np.ones(3, np.float32), ctx, 0.1)
    with pytest.raises(ValueError):
        M.discretization_count(np.zeros(2), np.ones(2), -1.0)
    q = np.array([0.5, -0.5], np.float32)
    from paper_2309_14545_b200 import Environment
    free = ValidationContext(rob.program, rob.model, rob.pairs, Environment())
    assert M.raked_motion_check(q, q, free, 0.05) == (True, 1)


def test_motion_repeated_calls_consistent(cuda):
    """Back-to-back launches (fresh and reused self-cleaning workspaces, PDL
    overlap of the begin, rake and finalize kernels) give identical results every time."""
    fx = golden_io.load("motion")
    key = "arm7_0"
    rob = load_robot("arm7")
    env = golden_io.env_from(fx, f"env_{key}")
    s, g, res = fx[f"starts_{key}"], fx[f"goals_{key}"], float(fx[f"res_{key}"])
    ws = runtime.motion_workspace(len(s))
    for rep in range(12):
        width = (8, 32, 1)[rep % 3]
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, env, width=width)
        b, n, blk = M.validate_motions(ctx, s, g, res, width=width, counts=True,
                                       workspace=ws if rep % 2 else None)
        assert runtime.unpack_bits(b.cpu().numpy(), len(s)).tolist() == \
            fx[f"verdict_{key}_w{width}_b0"].tolist()
        assert blk.cpu().numpy().tolist() == fx[f"blocks_{key}_w{width}_b0"].tolist()
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, env, width=8)
    for i in range(len(s)):
        assert M.raked_motion_check(s[i], g[i], ctx, res) == (
            bool(fx[f"verdict_{key}_w8_b0"][i]), int(fx[f"blocks_{key}_w8_b0"][i]))


@pytest.mark.parametrize("tiles", [1, 3, 17])   # 4,096 / 12,288 / 69,632 edges
def test_motion_batch_sizes_agree(cuda, tiles):
    """Batches of 1 / 3 / 17 copies of the config-2 edges (round 0 of one wave,
    of several waves per warp, and a queue far longer than the grid) give the verdicts,
    n and W-block counts of the oracle-checked 4,096-edge config 2 batch."""
    mw = workloads.config2()
    rob = load_robot("arm7")
    for width in (32, 8):
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env, width=width)
        ref = M.validate_motions(ctx, mw.starts, mw.goals, mw.resolution, width=width, counts=True)
        ref_v = runtime.unpack_bits(ref[0].cpu().numpy(), len(mw.starts))
        s, g = np.tile(mw.starts, (tiles, 1)), np.tile(mw.goals, (tiles, 1))
        ws = runtime.motion_workspace(len(s))
        for _ in range(2):                              # fresh, then reused workspace
            b, n, blk = M.validate_motions(ctx, s, g, mw.resolution, width=width, counts=True,
                                           workspace=ws)
            assert runtime.unpack_bits(b.cpu().numpy(), len(s)).tolist() == \
                np.tile(ref_v, tiles).tolist()
            assert n.cpu().numpy().tolist() == np.tile(ref[1].cpu().numpy(), tiles).tolist()
            assert blk.cpu().numpy().tolist() == np.tile(ref[2].cpu().numpy(), tiles).tolist()


def test_motion_sub_batches_above_4m_edges(cuda):
    """Above 2^22 edges vmp_validate_motions runs sub-batches on one workspace
    (csrc/vmp.cu): 1,025 copies of the config-2 edges give 1,025 copies of its
    verdicts, n and block counts."""
    torch = cuda
    mw = workloads.config2()
    rob = load_robot("arm7")
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
    ref = M.validate_motions(ctx, mw.starts, mw.goals, mw.resolution, counts=True)
    ref_v = runtime.unpack_bits(ref[0].cpu().numpy(), len(mw.starts))
    tiles = 1025
    s = torch.from_numpy(mw.starts).cuda().repeat(tiles, 1)
    g = torch.from_numpy(mw.goals).cuda().repeat(tiles, 1)
    assert len(s) > (1 << 22)
    b, n, blk = M.validate_motions(ctx, s, g, mw.resolution, counts=True)
    got = runtime.unpack_bits(b.cpu().numpy(), len(s)).reshape(tiles, -1)
    assert (got == ref_v[None, :]).all()
    assert (n.cpu().numpy().reshape(tiles, -1) == ref[1].cpu().numpy()[None, :]).all()
    assert (blk.cpu().numpy().reshape(tiles, -1) == ref[2].cpu().numpy()[None, :]).all()


def test_motion_very_long_edges_and_tiny_batches(cuda):
    """Very long edges (n up to ~57,000 states, ~1,800 chunks each) mixed with
    short ones, a zero-length edge, and batches of 0 / 1 edges - verdicts, n
    and W-lane block counts equal the dense oracle's.  Then six edges at
    1/65,536 rad: more chunks than the workspace has slots, so the owning warps
    finish the chunks that do not fit (the queue's overflow path)."""
    mw = workloads.config2()
    rob = load_robot("arm7")
    ob = O.Obstacles(mw.env.primitives)
    rng = np.random.default_rng(7)
    pick = rng.choice(len(mw.starts), 24, replace=False)
    s = mw.starts[pick].copy()
    g = mw.goals[pick].copy()
    g[3] = s[3]                                          # zero length: n = 1
    res = 1.0 / 8192.0                                   # n up to ~57,000 states
    ns = [O.discretization(a, b, res) for a, b in zip(s, g)]
    assert max(ns) > 32 * 1023
    states = [O.edge_all_states(rob.program, rob.pairs, ob, a, b, res)[1] for a, b in zip(s, g)]
    for width in (32, 8):
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env, width=width)
        bits, n, blk = M.validate_motions(ctx, s, g, res, width=width, counts=True)
        assert n.cpu().numpy().tolist() == ns
        for i, v in enumerate(states):
            ok, blocks = O.rake_blocks_from_states(v, width)
            assert bool(runtime.unpack_bits(bits.cpu().numpy(), len(s))[i]) == ok, i
            assert int(blk.cpu().numpy()[i]) == blocks, i
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
    empty = M.validate_motions(ctx, s[:0], g[:0], res)
    assert empty.numel() == 0
    one = M.validate_motions(ctx, s[:1], g[:1], res)
    assert bool(runtime.unpack_bits(one.cpu().numpy(), 1)[0]) == bool(states[0].all())
    # overflow: valid edges first, so their chunks are what the queue cannot hold
    order = np.argsort([not v.all() for v in states], kind="stable")[:6]
    s6, g6, fine = s[order], g[order], 1.0 / 65536.0
    n6 = [O.discretization(a, b, fine) for a, b in zip(s6, g6)]
    chunks = sum((n + 31) // 32 - 1 for n in n6)
    assert chunks > 8 * 8 + 32768, "need more chunks than slots (csrc/vmp.cu kDqSpareSlots)"
    st6 = [O.edge_all_states(rob.program, rob.pairs, ob, a, b, fine)[1] for a, b in zip(s6, g6)]
    bits, n, blk = M.validate_motions(ctx, s6, g6, fine, counts=True)
    assert n.cpu().numpy().tolist() == n6
    for i, v in enumerate(st6):
        ok, blocks = O.rake_blocks_from_states(v, 32)
        assert bool(runtime.unpack_bits(bits.cpu().numpy(), 6)[i]) == ok, i
        assert int(blk.cpu().numpy()[i]) == blocks, i


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4", "cfg5_16"])
def test_motion_other_robots_vs_oracle(cuda, cfg):
    """Raked motions of the fetch (8 joints, prismatic torso) and baxter (14
    joints, two arms) stand-ins in their config-3 / config-4 scenes (mixed
    spheres, capsules, cuboids; 64-65 obstacles, so two 32-obstacle broadphase
    chunks per kind run), and arm7 in the 16-primitive config-5 scene: verdicts,
    n and W-lane block counts (W = 32 and 8, forward and backward) equal the
    dense oracle's."""
    wl = workloads.config5(400, 16) if cfg == "cfg5_16" else \
        {"cfg3": workloads.config3, "cfg4": workloads.config4}[cfg](400)
    rob = load_robot(wl.robot)
    q = wl.q.T.copy()                                    # (400, dof)
    s, g = q[:200], q[200:]
    res = 1.0 / 16.0
    ob = O.Obstacles(wl.env.primitives)
    states = [O.edge_all_states(rob.program, rob.pairs, ob, a, b, res) for a, b in zip(s, g)]
    ns = [n for n, _ in states]
    assert 0 < np.mean([v.all() for _, v in states]) < 1
    for width in (32, 8):
        for bwd in (False, True):
            ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env, width=width)
            bits, n, blk = M.validate_motions(ctx, s, g, res, width=width, backward=bwd,
                                              counts=True)
            verdict = runtime.unpack_bits(bits.cpu().numpy(), len(s))
            assert n.cpu().numpy().tolist() == ns
            for i, (_, v) in enumerate(states):
                ok, blocks = O.rake_blocks_from_states(v, width, backward=bwd)
                assert bool(verdict[i]) == ok, (width, bwd, i)
                assert int(blk.cpu().numpy()[i]) == blocks, (width, bwd, i)
