"""Batched simplifier reproduces the reference's.

Golden runs of the reference shortcut / bspline_smooth / simplify_path
(simplify.py:61-118) on rrt_connect paths of the bundled problem sets, plus
two 80-waypoint zig-zag paths, are in tests/golden/simplify.npz
(make_simplify.py).  The speculative batching must return the identical
waypoints.  The CPU tests drive the speculation logic with the oracle's rake
(motion.py:38-78 restated) as the verdict source; the GPU tests run the
product path (device motion batches).
"""

import types

import numpy as np
import pytest

import golden_io
import vecmp_oracle as O
from paper_2309_14545_b200 import load_robot, simplify
from paper_2309_14545_b200.collision import ValidationContext
from paper_2309_14545_b200.simplify import Path, SimplifySettings

FX = golden_io.load("simplify")
KEYS = sorted(k[len("path_"):] for k in FX.files if k.startswith("path_"))
#: oracle-driven CPU cases: planar2 only (the numpy rake is ~100 edges/s for arm7)
CPU_KEYS = [k for k in KEYS if k.startswith("planar2")]


def _case(key):
    robot = load_robot(key.split("_", 1)[0])
    env = golden_io.env_from(FX, f"env_{key}")
    res, attempts, rounds, seed = FX[f"settings_{key}"]
    st = SimplifySettings(shortcut_attempts=int(attempts), smooth_rounds=int(rounds),
                          rng_seed=int(seed), resolution=float(res))
    return robot, env, st, Path(list(FX[f"path_{key}"]))


def _same(out, key, what):
    expect = FX[f"{what}_{key}"]
    got = np.stack(out.waypoints)
    assert got.shape == expect.shape, (key, what, got.shape, expect.shape)
    assert np.array_equal(got, expect), (key, what)


@pytest.fixture()
def oracle_verdicts(monkeypatch):
    """Replace the device batch with the oracle rake (verdicts and ctx.width-lane
    block counts), counting batches."""
    calls = []

    class OracleBatch(simplify._Batch):
        def __init__(self, ctx, starts, goals, resolution):
            calls.append(len(starts))
            self.ctx = ctx
            ob = O.Obstacles(ctx.env.primitives)
            res = [O.rake_check(ctx.program, ctx.pairs, ob, s, g, resolution, width=ctx.width)
                   for s, g in zip(starts, goals)]
            self.free = np.asarray([r[0] for r in res], dtype=bool)
            self.blocks = np.asarray([r[1] for r in res], dtype=np.int64)
    monkeypatch.setattr(simplify, "_Batch", OracleBatch)
    return calls


def _host_ctx(robot, env, width=8):
    return types.SimpleNamespace(program=robot.program, pairs=robot.pairs, env=env, width=width,
                                 motion_checks=0, blocks_evaluated=0)


def _counters(ctx, key, which):
    """ctx counters == the reference's for call `which` (0 shortcut, 1 smooth, 2 simplify)."""
    if f"counters_{key}" not in FX.files:
        return
    expect = FX[f"counters_{key}"][2 * which: 2 * which + 2].tolist()
    assert [ctx.motion_checks, ctx.blocks_evaluated] == expect, (key, which)


def _width(key):
    return int(FX[f"width_{key}"]) if f"width_{key}" in FX.files else 8


def test_settings_and_cost_mirror_reference():
    with pytest.raises(ValueError):
        SimplifySettings(shortcut_attempts=-1)
    with pytest.raises(ValueError):
        SimplifySettings(resolution=0.0)
    with pytest.raises(ValueError):
        simplify.path_cost(Path([np.zeros(2, np.float32)]))
    p = Path([np.asarray(v, np.float32) for v in ([0, 0], [3, 4], [3, 5])])
    assert simplify.path_cost(p) == pytest.approx(6.0)


def test_trivial_paths_are_identity(oracle_verdicts):
    robot = load_robot("planar2")
    ctx = _host_ctx(robot, golden_io.env_from(FX, f"env_{CPU_KEYS[0]}"))
    two = Path([np.zeros(2, np.float32), np.ones(2, np.float32)])
    assert np.array_equal(np.stack(simplify.shortcut(two, ctx, SimplifySettings()).waypoints),
                          np.stack(two.waypoints))
    three = Path([np.zeros(2, np.float32), np.asarray([1, 0], np.float32),
                  np.ones(2, np.float32)])
    out = simplify.bspline_smooth(three, ctx, SimplifySettings(smooth_rounds=0))
    assert np.array_equal(np.stack(out.waypoints), np.stack(three.waypoints))
    assert not oracle_verdicts


@pytest.mark.parametrize("key", CPU_KEYS)
def test_shortcut_speculation_matches_reference(oracle_verdicts, key):
    robot, env, st, path = _case(key)
    for spec in (1, 7, 32):
        ctx = _host_ctx(robot, env, _width(key))
        _same(simplify.shortcut(path, ctx, st, speculate=spec), key, "shortcut")
        _counters(ctx, key, 0)


@pytest.mark.parametrize("key", CPU_KEYS)
def test_smooth_chains_match_reference(oracle_verdicts, key):
    robot, env, st, path = _case(key)
    for window in (1, 5, 32):
        ctx = _host_ctx(robot, env, _width(key))
        _same(simplify.bspline_smooth(path, ctx, st, window=window), key, "smooth")
        _counters(ctx, key, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_simplify_on_device_matches_reference(cuda, key):
    robot, env, st, path = _case(key)
    for which, (what, fn) in enumerate((("shortcut", simplify.shortcut),
                                        ("smooth", simplify.bspline_smooth),
                                        ("simplify", simplify.simplify_path))):
        ctx = ValidationContext(robot.program, robot.model, robot.pairs, env, width=_width(key))
        _same(fn(path, ctx, st), key, what)
        _counters(ctx, key, which)
