"""Round-batched PRM reproduces the reference planner.

Golden runs of the reference prm (planners.py:243-291) on the bundled
problem sets are in tests/golden/prm.npz (make_golden.py); the batched
planner must return the identical waypoints after the identical number of
iterations, with three device launches per round instead of one call per
sample, per neighbour query and per edge.
"""

import time

import numpy as np
import pytest

import golden_io
from paper_2309_14545_b200 import load_robot
from paper_2309_14545_b200.prm import (HaltonDraws, PRMSettings, cheapest_route, prm_rounds,
                                       radical_inverse)

FX = golden_io.load("prm")
KEYS = sorted(k[len("start_"):] for k in FX.files if k.startswith("start_"))


def test_halton_and_route_helpers():
    assert radical_inverse(2, 1) == 0.5 and radical_inverse(3, 2) == 2.0 / 3.0
    d = HaltonDraws(np.array([[-1.0, 1.0], [0.0, 3.0]]))
    first = d.take(2)
    assert first.shape == (2, 2) and first.dtype == np.float32
    assert first[0].tolist() == [np.float32(0.0), np.float32(1.0)]
    adj = [[(2, 1.0), (3, 5.0)], [], [(1, 1.0)], [(1, 0.1)]]
    assert cheapest_route(adj, 0, 1) == [0, 2, 1]


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_prm_rounds_match_reference(cuda, key):
    robot = load_robot(key.split("_", 1)[0])
    env = golden_io.env_from(FX, f"env_{key}")
    res, max_it, k, batch, back, width = FX[f"settings_{key}"]
    settings = PRMSettings(resolution=float(res), max_iterations=int(max_it), prm_k=int(k),
                           prm_batch=int(batch), rake_backward=bool(back), width=int(width))
    t0 = time.perf_counter()
    out = prm_rounds(robot, env, FX[f"start_{key}"], FX[f"goal_{key}"], settings)
    seconds = time.perf_counter() - t0
    expect = FX[f"path_{key}"]
    assert out.success == (len(expect) > 0)
    assert out.iterations == int(FX[f"iterations_{key}"])
    assert np.array_equal(np.stack(out.waypoints), expect)
    assert out.device_calls <= 3 * out.rounds + 1
    # the reference's ValidationContext counters for the same run
    assert [out.blocks_evaluated, out.motion_checks] == FX[f"counters_{key}"].tolist()
    print(f"{key}: {seconds * 1e3:.1f} ms batched on the GPU vs "
          f"{float(FX[f'seconds_{key}']) * 1e3:.1f} ms reference (CPU)")
