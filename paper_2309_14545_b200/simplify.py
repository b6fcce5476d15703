"""Batched path post-processing over the B200 motion validator.

The reference simplifier (pkg/src/vecmp/simplify.py) is sequential: every
shortcut attempt and every smoothing proposal reads the path the previous one
left, and each asks ``validate_motion_rake`` one motion at a time.  Both loops
are rewritten here as speculation over the reference's own dependency
structure, so the returned waypoints are the reference's bit for bit while
the motion checks go to the device in batches:

* ``shortcut`` (simplify.py:61-94): the attempt sequence depends on the path
  only through the accepted splices.  Attempts are speculated in batches
  against the current path (the generator state before every attempt is
  kept); all their boundary/chord motions are validated in one launch and the
  attempts are replayed in order.  The first accepted splice rewinds the
  generator to the state after that attempt and the next batch starts from
  the new path - one launch per accepted splice plus one per ``speculate``
  rejected attempts.
* ``bspline_smooth`` (simplify.py:97-112): within a sweep, waypoint i's
  proposal depends on the already-updated waypoint i-1 and the old i, i+1.
  Whatever happened before i, the updated i-1 is either the old value (its
  proposal was rejected) or the proposal of the chain that started at the
  last rejection.  Every such chain over a window of ``window`` waypoints is
  computed on the host (the same float32 numpy expression), all their
  motions are validated in one launch, and the sweep then walks the chains -
  one launch per window per sweep instead of two motion calls per waypoint.

Proposal and splice arithmetic stays on the host with the reference's float32
expressions (it is O(D) per candidate; the rake is the work).  ``ctx`` may
be our ValidationContext or the reference's (motion._bind duck-types it);
``path`` may be our Path or the reference's - the result has the input's type.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import runtime
from .lanes import l2_distance
from .motion import _bind


@dataclass
class SimplifySettings:
    """Reference SimplifySettings (simplify.py:23-35): same fields, defaults, checks."""

    shortcut_attempts: int = 100
    smooth_rounds: int = 3
    rng_seed: int = 0
    resolution: float = 0.02

    def __post_init__(self) -> None:
        if self.shortcut_attempts < 0 or self.smooth_rounds < 0:
            raise ValueError("attempt and round counts must be non-negative")
        if self.resolution <= 0:
            raise ValueError("resolution must be positive")


@dataclass
class Path:
    """Waypoints from start to goal (reference planners.py:96-104)."""

    waypoints: list

    @property
    def cost(self) -> float:
        return float(sum(l2_distance(a, b) for a, b in zip(self.waypoints, self.waypoints[1:])))


def _waypoint_cost(waypoints) -> float:
    return float(sum(l2_distance(a, b) for a, b in zip(waypoints, waypoints[1:])))


def path_cost(path) -> float:
    """Sum of consecutive float32 distances (simplify.py:38-42)."""
    if len(path.waypoints) < 2:
        raise ValueError("a path needs at least two waypoints")
    return _waypoint_cost(path.waypoints)


def _cumulative_lengths(waypoints) -> np.ndarray:
    """Arc length at each waypoint (simplify.py:45-47)."""
    seg = [l2_distance(a, b) for a, b in zip(waypoints, waypoints[1:])]
    return np.concatenate([[0.0], np.cumsum(seg, dtype=np.float64)])


def _point_at(waypoints, cum: np.ndarray, u: float):
    """Segment index and float32 configuration at arc length u (simplify.py:50-58)."""
    seg = int(np.searchsorted(cum, u, side="right")) - 1
    seg = min(max(seg, 0), len(waypoints) - 2)
    length = cum[seg + 1] - cum[seg]
    t = 0.0 if length <= 0 else (u - cum[seg]) / length
    t32 = np.float32(min(max(t, 0.0), 1.0))
    a, b = waypoints[seg], waypoints[seg + 1]
    return seg, (a + t32 * (b - a)).astype(np.float32)


class _Batch:
    """Verdicts and ctx.width-lane rake block counts of speculated motions (one
    device launch).  The context's counters are NOT touched by the launch:
    ``charge(i)`` adds motion i exactly as the reference's sequential
    ``validate_motion_rake`` call would (motion.py:60 and one block per rake
    iteration), so after the replay ``ctx.motion_checks`` /
    ``ctx.blocks_evaluated`` equal the reference's."""

    def __init__(self, ctx, starts: list, goals: list, resolution: float):
        self.ctx = ctx
        self.free = np.zeros(0, dtype=bool)
        self.blocks = np.zeros(0, dtype=np.int64)
        if starts:
            sd = runtime.to_device(np.stack(starts))
            gd = runtime.to_device(np.stack(goals))
            words, _, blocks = runtime.validate_motions_device(
                *_bind(ctx), sd, gd, resolution, width=int(getattr(ctx, "width", 8)),
                prune=getattr(ctx, "prune", True), want_counts=True)
            self.free = runtime.unpack_bits(words.cpu().numpy(), len(starts))
            self.blocks = blocks.cpu().numpy().astype(np.int64)

    def charge(self, i: int) -> bool:
        self.ctx.motion_checks += 1
        self.ctx.blocks_evaluated += int(self.blocks[i])
        return bool(self.free[i])


def _like(path, waypoints):
    return type(path)(waypoints)


def shortcut(path, ctx, settings: SimplifySettings, *, speculate: int = 32):
    """Randomized shortcutting (simplify.py:61-94) with batched motion checks.

    Same generator stream, same candidate order and acceptance rule as the
    reference, so the output waypoints are identical.
    """
    waypoints = [np.asarray(w, dtype=np.float32).copy() for w in path.waypoints]
    if len(waypoints) <= 2 or settings.shortcut_attempts == 0:
        return _like(path, waypoints)
    speculate = max(1, int(speculate))
    rng = np.random.default_rng(settings.rng_seed)
    attempt = 0
    while attempt < settings.shortcut_attempts:
        cum = _cumulative_lengths(waypoints)
        total = float(cum[-1])
        if total <= 0:
            break
        stop = min(settings.shortcut_attempts, attempt + speculate)
        cands, after = [], []                  # (seg1, qa, seg2, qb) | None; rng state after
        starts, goals = [], []
        for _ in range(attempt, stop):
            u1, u2 = sorted(float(v) for v in rng.uniform(0.0, total, size=2))
            after.append(rng.bit_generator.state)
            seg1, qa = _point_at(waypoints, cum, u1)
            seg2, qb = _point_at(waypoints, cum, u2)
            if seg1 >= seg2 or (u2 - u1) - l2_distance(qa, qb) <= 1e-6:
                cands.append(None)
                continue
            cands.append((seg1, qa, seg2, qb))
            starts += [waypoints[seg1], qa, qb]
            goals += [qa, qb, waypoints[seg2 + 1]]
        batch = _Batch(ctx, starts, goals, settings.resolution)
        accepted = None
        m = 0
        for k, cand in enumerate(cands):
            if cand is None:
                continue
            # the reference checks the three motions in order and stops at the first failure
            ok = batch.charge(m) and batch.charge(m + 1) and batch.charge(m + 2)
            m += 3
            if not ok:
                continue
            seg1, qa, seg2, qb = cand
            spliced = waypoints[:seg1 + 1] + [qa, qb] + waypoints[seg2 + 1:]
            spliced = [w for i, w in enumerate(spliced)
                       if i == 0 or not np.array_equal(w, spliced[i - 1])]
            if _waypoint_cost(spliced) <= _waypoint_cost(waypoints):
                accepted = k
                waypoints = spliced
                break
        if accepted is None:
            attempt = stop
        else:
            attempt += accepted + 1
            rng.bit_generator.state = after[accepted]
    return _like(path, waypoints)


def _smooth_window(ctx, waypoints: list, lo: int, hi: int, resolution: float) -> None:
    """One sweep of simplify.py:105-110 over interior waypoints lo..hi-1, in place.

    Chain r (r = 0 .. hi-lo-1) starts at waypoint lo-1+r: for r = 0 with its
    already-final value, otherwise with its old value (its proposal was
    rejected); every later proposal of the chain is assumed accepted.  At
    step i the rows of ``heads`` are each live chain's value of waypoint i-1.
    """
    sixth = np.float32(1.0 / 6.0)
    four = np.float32(4.0)
    old = np.stack(waypoints[lo - 1:hi + 1])            # values of lo-1 .. hi on entry
    heads = old[0:1].copy()
    steps = []                                          # (heads, proposals, next) per i
    for i in range(lo, hi):
        cur, nxt = old[i - lo + 1], old[i - lo + 2]
        prop = ((heads + four * cur + nxt) * sixth).astype(np.float32)
        steps.append((heads, prop, nxt))
        heads = np.concatenate([prop, cur[None, :]], axis=0)
    starts = np.concatenate([np.concatenate([h, p]) for h, p, _ in steps])
    goals = np.concatenate([np.concatenate([p, np.broadcast_to(n, p.shape)])
                            for _, p, n in steps])
    batch = _Batch(ctx, list(starts), list(goals), resolution)
    live = pos = 0
    for i, (_, prop, _) in zip(range(lo, hi), steps):
        n = prop.shape[0]
        if batch.charge(pos + live) and batch.charge(pos + n + live):
            waypoints[i] = prop[live].copy()            # accepted: same chain continues
        else:
            live = n                                    # rejected: chain started at i
        pos += 2 * n


def bspline_smooth(path, ctx, settings: SimplifySettings, *, window: int = 32):
    """Iterated local cubic smoothing (simplify.py:97-112), one launch per
    ``window`` interior waypoints per sweep; output identical to the reference."""
    waypoints = [np.asarray(w, dtype=np.float32).copy() for w in path.waypoints]
    if len(waypoints) <= 2 or settings.smooth_rounds == 0:
        return _like(path, waypoints)
    window = max(1, int(window))
    last = len(waypoints) - 1
    for _ in range(settings.smooth_rounds):
        for lo in range(1, last, window):
            _smooth_window(ctx, waypoints, lo, min(last, lo + window), settings.resolution)
    return _like(path, waypoints)


def simplify_path(path, ctx, settings: SimplifySettings):
    """Shortcut then smooth (simplify.py:115-118)."""
    return bspline_smooth(shortcut(path, ctx, settings), ctx, settings)
