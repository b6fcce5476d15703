"""RRT-Connect with speculatively batched connect phases.

The reference (pkg/src/vecmp/planners.py:126-210) is sequential: every
iteration extends one tree toward a Halton sample (one rake-validated
motion), then greedily *connects* the other tree toward the new node - a
chain of ``_extend`` steps, each one nearest-neighbour query plus one motion
check, stopping at the first invalid motion.

The connect chain is determined before any of it is validated: from the
nearest node, every step moves ``range`` toward the same target, and the node
a step adds is strictly the closest to the target from then on (its distance
is below every distance seen before).  So the whole chain is computed on the
host with the reference's float32 expressions, its motions are validated in
ONE ``validate_motions`` launch, and the chain is replayed in order up to the
first invalid motion - identical tree, identical waypoints.  A step whose
newest node would not be strictly closest (never seen in practice) ends the
speculation and the next step re-queries the index, exactly as the reference.

Nearest-neighbour queries run on the device index (nn.NNIndex, exact, ties to
the first-inserted node); Halton draws reuse prm.HaltonDraws (bit-identical
to halton.py).  The reference's ValidationContext counters are reproduced:
one block per endpoint check, and for every motion the reference would have
validated (the walked prefix of each chain, including its failing motion)
one motion check and its W-lane rake block count.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import runtime
from .collision import ValidationContext
from .motion import validate_motions
from .nn import NNIndex
from .prm import HaltonDraws, InvalidProblemError

TRAPPED, ADVANCED, REACHED = range(3)


@dataclass
class RRTSettings:
    """The reference PlannerSettings fields RRT-Connect reads (planners.py:31-45)."""

    resolution: float = 0.02
    range: float = 2.0
    max_iterations: int = 1_000_000
    rake_backward: bool = False
    width: int = 8


@dataclass
class RRTResult:
    waypoints: list | None
    iterations: int
    blocks_evaluated: int = 0
    motion_checks: int = 0
    device_calls: int = 0

    @property
    def success(self) -> bool:
        return self.waypoints is not None


def _nn_dist(a: np.ndarray, b: np.ndarray) -> float:
    """NNIndex distance (nn.py:45-51): float32 squares summed in joint order."""
    d = (a - b).reshape(-1, 1)
    return float(np.sqrt(np.sum(d * d, axis=0, dtype=np.float32))[0])


def _step_toward(near: np.ndarray, target: np.ndarray, dist: float, rng: float):
    """The candidate of planners.py:158-163: (cand, reached)."""
    if dist <= rng:
        return target, True
    step = np.float32(rng / dist)
    return (near + step * (target - near)).astype(np.float32), False


class _Tree:
    """planners.py:129-150 with the device NN index."""

    def __init__(self, root: np.ndarray):
        self.configs = [root]
        self.parents = [-1]
        self.index = NNIndex(root.shape[0])
        self.index.insert(root, 0)

    def add(self, q: np.ndarray, parent: int) -> int:
        nid = len(self.configs)
        self.configs.append(q)
        self.parents.append(parent)
        self.index.insert(q, nid)
        return nid

    def chain(self, nid: int) -> list:
        out = []
        while nid >= 0:
            out.append(self.configs[nid])
            nid = self.parents[nid]
        out.reverse()
        return out


class _Planner:
    def __init__(self, ctx: ValidationContext, settings: RRTSettings, max_chain: int):
        self.ctx, self.s, self.max_chain = ctx, settings, max_chain
        self.blocks = 2                      # the two endpoint state_valid blocks
        self.checks = 0
        self.calls = 0

    def _validate(self, starts: list, goals: list):
        """Verdicts and W-lane block counts of a batch of motions (one launch)."""
        words, _, blk = validate_motions(self.ctx, np.stack(starts), np.stack(goals),
                                         self.s.resolution, backward=self.s.rake_backward,
                                         width=self.s.width, counts=True)
        self.calls += 1
        return (runtime.unpack_bits(words.cpu().numpy(), len(starts)), blk.cpu().numpy())

    def _account(self, blocks: np.ndarray, walked: int) -> None:
        self.checks += walked
        self.blocks += int(blocks[:walked].sum())

    def extend(self, tree: _Tree, target: np.ndarray):
        """planners.py:153-169."""
        near_id, dist = tree.index.nearest(target)
        near = tree.configs[near_id]
        if dist == 0.0:
            return REACHED, near_id
        cand, reached = _step_toward(near, target, dist, self.s.range)
        ok, blk = self._validate([near], [cand])
        self._account(blk, 1)
        if ok[0]:
            return (REACHED if reached else ADVANCED), tree.add(cand, near_id)
        return TRAPPED, -1

    def connect(self, tree: _Tree, target: np.ndarray) -> int:
        """planners.py:172-177, one launch per speculated chain."""
        while True:
            near_id, dist = tree.index.nearest(target)
            if dist == 0.0:
                return near_id
            # speculate: every step's nearest is the node the previous step added
            steps = []                       # (from, cand, reached, dist of cand or None)
            cur, d = tree.configs[near_id], dist
            while len(steps) < self.max_chain:
                cand, reached = _step_toward(cur, target, d, self.s.range)
                if reached:
                    steps.append((cur, cand, True))
                    break
                steps.append((cur, cand, False))
                d_next = _nn_dist(cand, target)
                if not d_next < d:           # the added node might not be the nearest
                    break
                cur, d = cand, d_next
                if d == 0.0:                 # next query is REACHED at this node
                    break
            ok, blk = self._validate([a for a, _, _ in steps], [b for _, b, _ in steps])
            parent = near_id
            for i, (_, cand, reached) in enumerate(steps):
                if not ok[i]:
                    self._account(blk, i + 1)
                    return -1
                parent = tree.add(cand, parent)
                if reached:
                    self._account(blk, i + 1)
                    return parent
            self._account(blk, len(steps))
            # chain ended without a verdict: the next step re-queries the index


def rrt_connect_batched(robot, env, start, goal, settings: RRTSettings | None = None, *,
                        max_chain: int = 4096) -> RRTResult:
    """Bidirectional RRT-Connect (planners.py:180-210) with batched connects."""
    settings = settings or RRTSettings()
    ctx = ValidationContext(robot.program, robot.model, robot.pairs, env, width=settings.width)
    start = np.asarray(start, dtype=np.float32).reshape(-1)
    goal = np.asarray(goal, dtype=np.float32).reshape(-1)
    ends = ctx.validate_configs(np.stack([start, goal], axis=1))
    if not ends[0]:
        raise InvalidProblemError("start configuration is in collision")
    if not ends[1]:
        raise InvalidProblemError("goal configuration is in collision")
    if np.array_equal(start, goal):
        return RRTResult([start.copy(), goal.copy()], 0, blocks_evaluated=2, device_calls=1)
    pl = _Planner(ctx, settings, max_chain)
    start_tree, goal_tree = _Tree(start), _Tree(goal)
    grow, other = start_tree, goal_tree
    draws = HaltonDraws(robot.limits)
    for iteration in range(1, settings.max_iterations + 1):
        sample = draws.take(1)[0]
        status, new_id = pl.extend(grow, sample)
        if status != TRAPPED:
            bridge = grow.configs[new_id]
            reached_id = pl.connect(other, bridge)
            if reached_id >= 0:
                if grow is start_tree:
                    forward, backward = grow.chain(new_id), other.chain(reached_id)
                else:
                    forward, backward = other.chain(reached_id), grow.chain(new_id)
                return RRTResult(forward + backward[::-1][1:], iteration, pl.blocks, pl.checks,
                                 pl.calls + 1)
        grow, other = other, grow
    return RRTResult(None, settings.max_iterations, pl.blocks, pl.checks, pl.calls + 1)
