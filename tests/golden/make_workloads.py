"""Generate the config-2 motion workload (4,096 arm7 edges) - run once, committed.

BASELINE config 2: endpoints uniform in the joint limits; about half the
edges forced collision-free; resolution 1/32; 24 cuboids + 8 capsules with
the keep-out rule (paper_2309_14545_b200.workloads.config2_scene).

Forcing edges free needs a validator, so the edge set is generated here on
the CPU with the oracle (test infrastructure) and committed as
paper_2309_14545_b200/data/cfg2_edges.npz; the benchmark arms and the tests
then load the identical endpoints.  Procedure: even-indexed
edges resample the start until it is valid, then the goal until the rake
verdict of the whole edge is valid; odd-indexed edges are plain uniform.

    python tests/golden/make_workloads.py
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import vecmp_oracle as O  # noqa: E402
from paper_2309_14545_b200 import load_robot, workloads  # noqa: E402

N_EDGES = 4096
SEED = 2


def main() -> None:
    rob = load_robot("arm7")
    env = workloads.config2_scene()
    ob = O.Obstacles(env.primitives)
    lims = rob.limits
    rng = np.random.default_rng(SEED)
    res = workloads.CFG2_RESOLUTION

    def draw():
        return rng.uniform(lims[:, 0], lims[:, 1]).astype(np.float32)

    def state_ok(q):
        return bool(O.validate_lanes(rob.program, rob.pairs, ob, q.reshape(-1, 1), prune=False)[0])

    starts = np.empty((N_EDGES, 7), np.float32)
    goals = np.empty((N_EDGES, 7), np.float32)
    attempts = 0
    for e in range(N_EDGES):
        s, g = draw(), draw()
        if e % 2 == 0:
            while not state_ok(s):
                s = draw()
            while True:
                attempts += 1
                _, valid = O.edge_all_states(rob.program, rob.pairs, ob, s, g, res)
                if valid.all():
                    break
                g = draw()
        starts[e], goals[e] = s, g
    out = ROOT / "paper_2309_14545_b200" / "data" / "cfg2_edges.npz"
    out.parent.mkdir(exist_ok=True)
    np.savez_compressed(out, starts=starts, goals=goals, resolution=np.float64(res),
                        seed=np.int64(SEED))
    print(f"wrote {out} ({N_EDGES} edges, {attempts} forced-free attempts)")


if __name__ == "__main__":
    main()
