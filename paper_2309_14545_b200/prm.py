"""Round-batched incremental PRM over the B200 validators.

The reference PRM (pkg/src/vecmp/planners.py:243-291) draws ``prm_batch``
Halton samples per round, checks each with ``ctx.state_valid`` and each of its
``prm_k`` nearest-vertex edges with ``validate_motion_rake``, one call at a
time.  Validity is order-independent, so a round maps onto three device calls:

1. every sample of the round in one ``validate_batch`` launch;
2. the k nearest vertices of every valid sample in one exact k-NN launch
   (nn.NNIndex.k_nearest_many); sample j only sees the vertices inserted
   before it - the ones before the round plus the valid samples before j -
   exactly as the reference's insert-after-query loop;
3. the k-NN edges of all valid samples in one ``validate_motions`` launch.

Vertices, adjacency lists and the shortest-path query are then updated in
the reference's order, so the roadmap - and the returned waypoints - are the
reference's whenever the verdicts are (tests/test_gpu_prm.py checks the
waypoints against the reference's own runs).

Host helpers restated from the reference: Halton draws (halton.py:17-67),
uniform-cost search (planners.py:213-240).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

from . import runtime
from .collision import ValidationContext
from .motion import validate_motions
from .nn import NNIndex


def halton_bases(count: int) -> list[int]:
    bases: list[int] = []
    n = 2
    while len(bases) < count:
        if all(n % b for b in bases):
            bases.append(n)
        n += 1
    return bases


def radical_inverse(base: int, index: int) -> float:
    """Base-``base`` digit reversal of ``index`` (same float64 accumulation
    order as reference halton.py:27-40, so draws are bit-identical)."""
    step = 1.0 / base
    scale = step
    acc = 0.0
    while index > 0:
        index, digit = divmod(index, base)
        acc += digit * scale
        scale *= step
    return acc


class HaltonDraws:
    """Halton sequence scaled to joint limits, index starting at 1."""

    def __init__(self, limits: np.ndarray):
        self.lo = np.asarray(limits, dtype=np.float64)[:, 0]
        self.hi = np.asarray(limits, dtype=np.float64)[:, 1]
        self.bases = halton_bases(len(self.lo))
        self.index = 1

    def take(self, count: int) -> np.ndarray:
        """(count, dof) float32 - the next ``count`` draws."""
        out = np.empty((count, len(self.lo)), dtype=np.float32)
        for r in range(count):
            u = np.asarray([radical_inverse(b, self.index) for b in self.bases])
            out[r] = (self.lo + u * (self.hi - self.lo)).astype(np.float32)
            self.index += 1
        return out


def cheapest_route(adjacency: list, source: int, target: int) -> list[int] | None:
    """Uniform-cost search; equal-cost ties resolved by heap order on (cost, vertex)."""
    best = [float("inf")] * len(adjacency)
    parent = [-1] * len(adjacency)
    closed = [False] * len(adjacency)
    best[source] = 0.0
    frontier = [(0.0, source)]
    while frontier:
        cost, v = heapq.heappop(frontier)
        if closed[v]:
            continue
        closed[v] = True
        if v == target:
            route = []
            while v >= 0:
                route.append(v)
                v = parent[v]
            return route[::-1]
        for u, w in adjacency[v]:
            c = cost + w
            if c < best[u]:
                best[u], parent[u] = c, v
                heapq.heappush(frontier, (c, u))
    return None


@dataclass
class PRMSettings:
    """The reference PlannerSettings fields PRM reads (planners.py:31-45)."""

    resolution: float = 0.02
    max_iterations: int = 1_000_000
    prm_k: int = 8
    prm_batch: int = 128
    rake_backward: bool = False
    width: int = 8


class InvalidProblemError(ValueError):
    """Start or goal rejected at setup (reference planners.py:27-28)."""


@dataclass
class PRMResult:
    waypoints: list | None
    iterations: int
    rounds: int
    device_calls: int
    #: the reference's ValidationContext counters for the same run: one block
    #: per state_valid (endpoints + samples) plus the W-lane rake blocks of
    #: every edge; one motion check per edge (collision.py:453-465, motion.py:60)
    blocks_evaluated: int = 0
    motion_checks: int = 0

    @property
    def success(self) -> bool:
        return self.waypoints is not None


def prm_rounds(robot, env, start, goal, settings: PRMSettings | None = None) -> PRMResult:
    """Incremental PRM with one state-validity launch and one motion launch per round."""
    settings = settings or PRMSettings()
    ctx = ValidationContext(robot.program, robot.model, robot.pairs, env, width=settings.width)
    start = np.asarray(start, dtype=np.float32).reshape(-1)
    goal = np.asarray(goal, dtype=np.float32).reshape(-1)
    ends = ctx.validate_configs(np.stack([start, goal], axis=1))
    if not ends[0]:
        raise InvalidProblemError("start configuration is in collision")
    if not ends[1]:
        raise InvalidProblemError("goal configuration is in collision")
    if np.array_equal(start, goal):
        return PRMResult([start.copy(), goal.copy()], 0, 0, 1, blocks_evaluated=2)
    vertices = [start, goal]
    adjacency: list[list[tuple[int, float]]] = [[], []]
    nn = NNIndex(len(start))
    nn.insert(start, 0)
    nn.insert(goal, 1)
    draws = HaltonDraws(robot.limits)
    iterations = rounds = calls = 0
    blocks, checks = 2, 0                  # endpoint state_valid blocks
    calls += 1
    while iterations < settings.max_iterations:
        count = min(settings.prm_batch, settings.max_iterations - iterations)
        samples = draws.take(count)
        iterations += count
        rounds += 1
        ok = ctx.validate_configs(np.ascontiguousarray(samples.T))       # launch 1
        calls += 1
        edges = []                                                         # (vid, nbr, dist)
        fresh = samples[ok]
        if len(fresh):
            # sample j of the round sees the vertices inserted before it
            base = len(vertices)
            nn.insert_many(fresh, range(base, base + len(fresh)))
            nbr, dist = nn.k_nearest_many(fresh, settings.prm_k,                # launch 2
                                          visible=base + np.arange(len(fresh)))
            calls += 1
            for j, sample in enumerate(fresh):
                vertices.append(sample)
                adjacency.append([])
                edges.extend((base + j, int(b), float(d)) for b, d in zip(nbr[j], dist[j])
                             if b >= 0)
        if edges:
            starts = np.stack([vertices[nbr] for _, nbr, _ in edges])
            goals = np.stack([vertices[vid] for vid, _, _ in edges])
            words, _, nblk = validate_motions(ctx, starts, goals, settings.resolution,  # launch 3
                                              backward=settings.rake_backward,
                                              width=settings.width, counts=True)
            calls += 1
            blocks += int(nblk.sum())
            checks += len(edges)
            free = runtime.unpack_bits(words.cpu().numpy(), len(edges))
            for (vid, nbr, dist), edge_ok in zip(edges, free):
                if edge_ok:
                    adjacency[nbr].append((vid, dist))
                    adjacency[vid].append((nbr, dist))
        route = cheapest_route(adjacency, 0, 1)
        if route is not None:
            return PRMResult([vertices[v] for v in route], iterations, rounds, calls,
                             blocks + iterations, checks)
    return PRMResult(None, iterations, rounds, calls, blocks + iterations, checks)
