"""RRT-Connect with batched connect chains reproduces
the reference planner.

tests/golden/rrt.npz holds the reference rrt_connect's runs (planners.py:
180-210) on the bundled problem sets and on arm7 in the config-2 clutter
(make_rrt.py): waypoints, iteration counts and ValidationContext counters.
The CPU tests drive the speculation logic with oracle verdicts / W-block
counts and a host k-NN restatement; the GPU tests run the product path.
"""

import numpy as np
import pytest

import golden_io
import vecmp_oracle as O
from paper_2309_14545_b200 import load_robot, rrt
from paper_2309_14545_b200.rrt import RRTSettings, rrt_connect_batched

FX = golden_io.load("rrt")
KEYS = sorted(k[len("start_"):] for k in FX.files if k.startswith("start_"))
CPU_KEYS = [k for k in KEYS if not k.startswith("arm7_clutter")]


def _case(key):
    robot = load_robot(key.split("_", 1)[0])
    env = golden_io.env_from(FX, f"env_{key}")
    res, rng, max_it, back, width = FX[f"settings_{key}"]
    st = RRTSettings(resolution=float(res), range=float(rng), max_iterations=int(max_it),
                     rake_backward=bool(back), width=int(width))
    return robot, env, st


def _check(out, key):
    expect = FX[f"path_{key}"]
    assert out.success == (len(expect) > 0)
    assert out.iterations == int(FX[f"iterations_{key}"])
    assert np.array_equal(np.stack(out.waypoints), expect)
    assert [out.blocks_evaluated, out.motion_checks] == FX[f"counters_{key}"].tolist()


class _HostNN:
    """Oracle restatement of nn.py (test infrastructure only)."""

    def __init__(self, dim):
        self.pts = np.empty((dim, 0), np.float32)

    def insert(self, q, payload):
        self.pts = np.concatenate([self.pts, np.asarray(q, np.float32).reshape(-1, 1)], axis=1)

    def nearest(self, q):
        idx, dist = O.nn_k_nearest(self.pts, q, 1)
        return int(idx[0]), float(dist[0])


@pytest.fixture()
def oracle_planner(monkeypatch):
    def validate(self, starts, goals):
        ob = O.Obstacles(self.ctx.env.primitives)
        res = [O.rake_check(self.ctx.program, self.ctx.pairs, ob, s, g, self.s.resolution,
                            width=self.s.width, backward=self.s.rake_backward)
               for s, g in zip(starts, goals)]
        self.calls += 1
        return np.asarray([v for v, _ in res]), np.asarray([b for _, b in res])
    monkeypatch.setattr(rrt._Planner, "_validate", validate)
    monkeypatch.setattr(rrt, "NNIndex", _HostNN)
    monkeypatch.setattr(rrt, "ValidationContext", _HostCtx)


class _HostCtx:
    def __init__(self, program, model, pairs, env, width=8):
        self.program, self.pairs, self.env = program, pairs, env

    def validate_configs(self, q):
        return O.validate_configs(self.program, self.pairs, self.env.primitives, q)


@pytest.mark.parametrize("key", CPU_KEYS)
def test_connect_speculation_matches_reference(oracle_planner, key):
    robot, env, st = _case(key)
    for max_chain in (1, 3, 4096):
        _check(rrt_connect_batched(robot, env, FX[f"start_{key}"], FX[f"goal_{key}"], st,
                                   max_chain=max_chain), key)


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_rrt_connect_on_device_matches_reference(cuda, key):
    robot, env, st = _case(key)
    out = rrt_connect_batched(robot, env, FX[f"start_{key}"], FX[f"goal_{key}"], st)
    _check(out, key)
    # one launch per extend and per connect chain, never one per motion
    assert out.device_calls <= 2 * out.iterations + 2
