"""CPU ORACLE for the FK -> collision check -> raked motion validation path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs may import this module,
and only as the checker or as the timed CPU baseline - never as part of the
product path (paper_2309_14545_b200/ never imports it).

What it is: a NumPy restatement of the reference algorithm (arxiv 2309.14545
package ``vecmp``, pure Python/NumPy; numpy pinned ``>=1.24`` in
pkg/pyproject.toml:10-13, 2.3.5 here) that reproduces its float32 results bit
for bit, plus a new float64 signed-clearance oracle that classifies the
+-1e-4 m verdict band (the reference computes no distances).

Pinned against the reference itself: tests/golden/make_golden.py imports the
reference from /root/reference (this container only) and records programs,
FK rows, block verdicts (W = 8, prune on/off, reject_all), rake verdicts and
block counts, discretisation counts and narrowphase cases;
tests/test_oracle_golden.py checks this module reproduces every one.

Reference functions restated (file:line in /root/reference/pkg/src/vecmp):
  f32 lane interpreter           program.py:157-214
  packed obstacles / thresholds  collision.py:57-103
  sphere / capsule / box hits    collision.py:206-254
  BlockValidator state machine   collision.py:293-408 (coarse "any lane"
                                 prune, fine OR, self pairs, abort)
  validate_block                 collision.py:411-430
  l2_distance, discretization    lanes.py:106-113, motion.py:25-29
  interpolate_lanes, rake        lanes.py:91-103, motion.py:32-78
  float64 FK                     trace.py:100-137 (graph semantics)
  float64 distance oracles       pkg/tests/test_collision.py:24-39,136-159
  exact k-NN scan                nn.py:45-69 (float32 joint-order sum, stable
                                 argsort: ties to the first-inserted point)
"""

from __future__ import annotations

import math

import numpy as np

CONST, INPUT, ADD, SUB, MUL, NEG, SIN, COS = range(8)
F32 = np.float32


# ------------------------------------------------------------------ programs

class _Feed:
    """Per-program op tuples, split into const rows and dynamic ops."""

    def __init__(self, program):
        kinds = [int(k) for k in program.kinds]
        self.n = len(kinds)
        self.consts = [(i, float(program.values[i])) for i, k in enumerate(kinds) if k == CONST]
        self.ops = [(i, k, int(program.a[i]), int(program.b[i]), float(program.values[i]))
                    for i, k in enumerate(kinds) if k != CONST]
        self.markers = list(program.checks)


_FEEDS: dict = {}


def _feed(program) -> _Feed:
    f = _FEEDS.get(id(program))
    if f is None or f[0] is not program:
        f = _FEEDS[id(program)] = (program, _Feed(program))
    return f[1]


def rows_f32(program, data: np.ndarray) -> np.ndarray:
    """All op rows in float32, one numpy ufunc per op (program.py:175-208)."""
    fd = _feed(program)
    data = np.asarray(data, dtype=F32)
    rows = np.empty((fd.n, data.shape[1]), dtype=F32)
    for i, v in fd.consts:
        rows[i] = F32(v)
    for i, k, a, b, v in fd.ops:
        if k == MUL:
            np.multiply(rows[a], rows[b], out=rows[i])
        elif k == ADD:
            np.add(rows[a], rows[b], out=rows[i])
        elif k == SUB:
            np.subtract(rows[a], rows[b], out=rows[i])
        elif k == SIN:
            np.sin(rows[a], out=rows[i])
        elif k == COS:
            np.cos(rows[a], out=rows[i])
        elif k == NEG:
            np.negative(rows[a], out=rows[i])
        else:
            rows[i] = data[int(v)]
    return rows


def rows_f64(program, q: np.ndarray) -> np.ndarray:
    """Float64 evaluation of the same op list (= evaluate_graph semantics)."""
    fd = _feed(program)
    q = np.asarray(q, dtype=np.float64)          # (dof, N)
    rows = np.empty((fd.n, q.shape[1]), dtype=np.float64)
    for i, v in fd.consts:
        rows[i] = v
    for i, k, a, b, v in fd.ops:
        if k == MUL:
            np.multiply(rows[a], rows[b], out=rows[i])
        elif k == ADD:
            np.add(rows[a], rows[b], out=rows[i])
        elif k == SUB:
            np.subtract(rows[a], rows[b], out=rows[i])
        elif k == SIN:
            np.sin(rows[a], out=rows[i])
        elif k == COS:
            np.cos(rows[a], out=rows[i])
        elif k == NEG:
            np.negative(rows[a], out=rows[i])
        else:
            rows[i] = q[int(v)]
    return rows


def marker_centres(program, rows: np.ndarray) -> np.ndarray:
    """(n_markers, 3, N) centres gathered from op rows."""
    idx = np.asarray([m.xyz for m in program.checks], dtype=np.int64).reshape(-1, 3)
    return rows[idx]


# ----------------------------------------------------------------- obstacles

def _kind(p) -> str:
    if hasattr(p, "p0"):
        return "capsule"
    if hasattr(p, "half_extents"):
        return "box"
    return "sphere"


class Obstacles:
    """float32 SoA obstacle arrays grouped by kind (collision.py:57-103)."""

    def __init__(self, primitives):
        sph = [p for p in primitives if _kind(p) == "sphere"]
        cap = [p for p in primitives if _kind(p) == "capsule"]
        box = [p for p in primitives if _kind(p) == "box"]
        self.sc = np.asarray([p.center for p in sph], dtype=F32).reshape(-1, 3)
        self.sr = np.asarray([p.radius for p in sph], dtype=F32)
        self.cp0 = np.asarray([p.p0 for p in cap], dtype=F32).reshape(-1, 3)
        ax64 = np.asarray([np.asarray(p.p1, float) - np.asarray(p.p0, float) for p in cap],
                          dtype=np.float64).reshape(-1, 3)
        vv = (ax64 * ax64).sum(axis=1)
        safe = np.maximum(vv, 1e-300)
        self.cax = ax64.astype(F32)
        self.cinv = np.where(vv > 1e-18, 1.0 / safe, 0.0).astype(F32)
        self.cr = np.asarray([p.radius for p in cap], dtype=F32)
        self.bc = np.asarray([p.center for p in box], dtype=F32).reshape(-1, 3)
        self.bh = np.asarray([p.half_extents for p in box], dtype=F32).reshape(-1, 3)
        rt = np.asarray([np.asarray(p.rotation, float).T for p in box], dtype=F32).reshape(-1, 3, 3)
        # per-(row, col) contiguous columns ready to broadcast against lanes
        self.bcols = [np.ascontiguousarray(rt[:, i, j])[:, None] for i in range(3) for j in range(3)]
        self.bhi = [np.ascontiguousarray(self.bh[:, i])[:, None] for i in range(3)]
        self.blo = [-c for c in self.bhi]
        self.primitives = list(primitives)
        self._memo: dict = {}

    @property
    def sizes(self) -> tuple[int, int, int]:
        return len(self.sr), len(self.cr), len(self.bh)

    def sphere_thr(self, r: float) -> np.ndarray:
        key = ("s", r)
        if key not in self._memo:
            self._memo[key] = (self.sr + F32(r)) ** 2
        return self._memo[key]

    def capsule_thr(self, r: float) -> np.ndarray:
        key = ("c", r)
        if key not in self._memo:
            self._memo[key] = (self.cr + F32(r)) ** 2
        return self._memo[key]


def hits_spheres(centres, thr, pos) -> np.ndarray:
    """(K, W) contact of lane positions pos (3, W) against sphere centres."""
    d = centres[:, :, None] - pos[None, :, :]
    np.multiply(d, d, out=d)
    acc = d[:, 0] + d[:, 1]
    acc += d[:, 2]
    return acc <= thr[:, None]


def hits_capsules(p0, axis, inv, thr, pos) -> np.ndarray:
    d = pos[None, :, :] - p0[:, :, None]
    t = d[:, 0] * axis[:, 0, None]
    t += d[:, 1] * axis[:, 1, None]
    t += d[:, 2] * axis[:, 2, None]
    t *= inv[:, None]
    np.minimum(t, F32(1.0), out=t)
    np.maximum(t, F32(0.0), out=t)
    d -= t[:, None, :] * axis[:, :, None]
    np.multiply(d, d, out=d)
    acc = d[:, 0] + d[:, 1]
    acc += d[:, 2]
    return acc <= thr[:, None]


def hits_boxes(centre, cols, hi, lo, pos, radius: float) -> np.ndarray:
    d = pos[None, :, :] - centre[:, :, None]
    total = None
    for axis in range(3):
        loc = cols[3 * axis] * d[:, 0]
        loc += cols[3 * axis + 1] * d[:, 1]
        loc += cols[3 * axis + 2] * d[:, 2]
        cl = np.minimum(loc, hi[axis])
        np.maximum(cl, lo[axis], out=cl)
        loc -= cl
        np.multiply(loc, loc, out=loc)
        total = loc if total is None else total + loc
    return total <= F32(radius) ** 2


def _box_sel(ob: Obstacles, sel):
    if sel is None:
        return ob.bc, ob.bcols, ob.bhi, ob.blo
    return (ob.bc[sel], [c[sel] for c in ob.bcols], [c[sel] for c in ob.bhi],
            [c[sel] for c in ob.blo])


def kind_hits(ob: Obstacles, pos: np.ndarray, radius: float, sel=(None, None, None)):
    """Per-kind (K, W) contact matrices (None for an empty kind / empty selection)."""
    ss, cs, bs = sel
    out = []
    if len(ob.sr) and (ss is None or len(ss)):
        c = ob.sc if ss is None else ob.sc[ss]
        t = ob.sphere_thr(radius) if ss is None else ob.sphere_thr(radius)[ss]
        out.append(hits_spheres(c, t, pos))
    else:
        out.append(None)
    if len(ob.cr) and (cs is None or len(cs)):
        args = (ob.cp0, ob.cax, ob.cinv, ob.capsule_thr(radius))
        if cs is not None:
            args = tuple(a[cs] for a in args)
        out.append(hits_capsules(*args, pos))
    else:
        out.append(None)
    if len(ob.bh) and (bs is None or len(bs)):
        out.append(hits_boxes(*_box_sel(ob, bs), pos, radius))
    else:
        out.append(None)
    return out


# ------------------------------------------------------------ block verdicts

def _partners(pairs) -> dict:
    table: dict = {}
    for a, b in pairs.pairs:
        lo, hi = min(a, b), max(a, b)
        table.setdefault(hi, []).append(lo)
    for v in table.values():
        v.sort()
    return table


def validate_lanes(program, pairs, ob: Obstacles, data: np.ndarray, *, prune: bool = True,
                   reject_all: bool = False, rows: np.ndarray | None = None) -> np.ndarray:
    """Per-lane validity of one block (collision.py:293-430); True = VALID.

    Markers stream in program order; coarse markers compute the "any lane"
    active obstacle sets, fine markers OR environment contacts and test self
    pairs, and the walk aborts when no lane (reject_all: not every lane)
    remains valid.
    """
    if rows is None:
        rows = rows_f32(program, data)
    width = rows.shape[1]
    valid = np.ones(width, dtype=bool)
    partners = _partners(pairs)
    seen: dict = {}
    active: dict = {}
    for m in program.checks:
        pos = np.empty((3, width), dtype=F32)
        pos[0], pos[1], pos[2] = rows[m.xyz[0]], rows[m.xyz[1]], rows[m.xyz[2]]
        if m.level == "coarse":
            if prune:
                sets = []
                for h in kind_hits(ob, pos, m.radius):
                    if h is None:
                        sets.append(None)
                        continue
                    anyl = h.any(axis=1)
                    sets.append(None if anyl.all() else np.flatnonzero(anyl))
                active[m.link] = tuple(sets)
            continue
        sel = active.get(m.link, (None, None, None)) if prune else (None, None, None)
        collide = None
        for h in kind_hits(ob, pos, m.radius, sel):
            if h is not None:
                hit = h.any(axis=0)
                collide = hit if collide is None else (collide | hit)
        changed = False
        if collide is not None and collide.any():
            valid &= ~collide
            changed = True
        for lo in partners.get(m.link, ()):
            for px, py, pz, pr in seen.get(lo, ()):
                dx, dy, dz = pos[0] - px, pos[1] - py, pos[2] - pz
                thr = F32(m.radius + pr) ** 2
                clear = dx * dx + dy * dy + dz * dz > thr
                if not clear.all():
                    valid &= clear
                    changed = True
        if partners:
            seen.setdefault(m.link, []).append((pos[0].copy(), pos[1].copy(), pos[2].copy(),
                                                m.radius))
        if changed and ((reject_all and not valid.all()) or not valid.any()):
            break
    if reject_all and not valid.all():
        return np.zeros(width, dtype=bool)
    return valid


def validate_configs(program, pairs, primitives, q: np.ndarray, *, prune: bool = False,
                     chunk: int = 65536) -> np.ndarray:
    """Verdicts of a (dof, N) batch, processed as wide blocks (width-independent)."""
    ob = primitives if isinstance(primitives, Obstacles) else Obstacles(primitives)
    q = np.asarray(q, dtype=F32)
    n = q.shape[1]
    out = np.empty(n, dtype=bool)
    for s in range(0, n, chunk):
        blk = q[:, s:s + chunk]
        out[s:s + blk.shape[1]] = validate_lanes(program, pairs, ob, blk, prune=prune)
    return out


# ------------------------------------------------------- float64 clearances

def _seg_dist(p, a, b):
    ab = b - a
    denom = float(ab @ ab)
    rel = p - a[:, None]
    if denom == 0.0:
        t = np.zeros(p.shape[1])
    else:
        t = np.clip((ab @ rel) / denom, 0.0, 1.0)
    close = a[:, None] + t[None, :] * ab[:, None]
    return np.linalg.norm(p - close, axis=0)


def _box_dist(p, centre, half, rot):
    local = rot.T @ (p - centre[:, None])
    clamped = np.clip(local, -half[:, None], half[:, None])
    return np.linalg.norm(local - clamped, axis=0)


def primitive_gap_f64(p, c: np.ndarray, radius: float) -> np.ndarray:
    """float64 signed gap between spheres of ``radius`` at points c (3, n) and
    one primitive (closest-point forms of pkg/tests/test_collision.py:24-39)."""
    kind = _kind(p)
    if kind == "sphere":
        d = np.linalg.norm(c - np.asarray(p.center, float)[:, None], axis=0)
        return d - (float(p.radius) + radius)
    if kind == "capsule":
        return _seg_dist(c, np.asarray(p.p0, float), np.asarray(p.p1, float)) \
            - (float(p.radius) + radius)
    return _box_dist(c, np.asarray(p.center, float), np.asarray(p.half_extents, float),
                     np.asarray(p.rotation, float)) - radius


def clearance_f64(program, pairs, primitives, q: np.ndarray) -> np.ndarray:
    """Minimum signed clearance (m) per configuration, float64.

    Fine-sphere centres come from the float64 program evaluation at the
    float32 inputs; distances follow the closest-point forms of
    pkg/tests/test_collision.py:24-39 and the pair set of :136-159.
    clearance <= 0  <=>  the float64 semantics say "in collision".
    """
    q64 = np.asarray(q, dtype=F32).astype(np.float64)
    rows = rows_f64(program, q64)
    fine = [m for m in program.checks if m.level == "fine"]
    n = q64.shape[1]
    best = np.full(n, np.inf)
    cen = {}
    for m in fine:
        c = rows[list(m.xyz)]
        cen.setdefault(m.link, []).append((c, m.radius))
        for p in primitives:
            np.minimum(best, primitive_gap_f64(p, c, m.radius), out=best)
    for a, b in pairs.pairs:
        for ca, ra in cen.get(a, ()):
            for cb, rb in cen.get(b, ()):
                gap = np.linalg.norm(ca - cb, axis=0) - (ra + rb)
                np.minimum(best, gap, out=best)
    return best


# --------------------------------------------------------------- motions

def np_l2(a, b) -> float:
    x = np.asarray(a, dtype=F32).reshape(-1)
    y = np.asarray(b, dtype=F32).reshape(-1)
    d = x - y
    return float(np.sqrt(np.sum(d * d, dtype=F32)))


def discretization(start, goal, resolution: float) -> int:
    if resolution <= 0:
        raise ValueError(f"resolution must be positive, got {resolution}")
    return max(1, math.ceil(np_l2(start, goal) / resolution))


def rake_states(start, goal, n: int, indices: np.ndarray) -> np.ndarray:
    """(dof, len(indices)) states at t = f32(i / n), unfused float32 lerp."""
    s = np.asarray(start, dtype=F32).reshape(-1)
    g = np.asarray(goal, dtype=F32).reshape(-1)
    t = (np.asarray(indices, dtype=np.int64) / n).astype(F32)
    return s[:, None] + t[None, :] * (g - s)[:, None]


def rake_check(program, pairs, ob: Obstacles, start, goal, resolution: float, width: int = 8,
               backward: bool = False, prune: bool = True) -> tuple[bool, int]:
    """Stratified rake, one W-lane block per iteration (motion.py:38-78)."""
    n = discretization(start, goal, resolution)
    s = math.ceil(n / width)
    bases = np.arange(width, dtype=np.int64) * s
    order = range(s, 0, -1) if backward else range(1, s + 1)
    blocks = 0
    for j in order:
        idx = bases + j
        inr = idx <= n
        data = rake_states(start, goal, n, np.where(inr, idx, idx[0]))
        ok = validate_lanes(program, pairs, ob, data, prune=prune)
        blocks += 1
        if not ok[inr].all():
            return False, blocks
    return True, blocks


def edge_all_states(program, pairs, ob: Obstacles, start, goal, resolution: float):
    """(n, per-state validity in index order 1..n) - dense, for fixtures and bands."""
    n = discretization(start, goal, resolution)
    idx = np.arange(1, n + 1, dtype=np.int64)
    data = rake_states(start, goal, n, idx)
    return n, validate_lanes(program, pairs, ob, data, prune=False)


def rake_blocks_from_states(valid: np.ndarray, width: int, backward: bool = False) -> tuple[bool, int]:
    """Verdict and W-rake block count implied by per-state validity (index order)."""
    n = len(valid)
    s = math.ceil(n / width)
    bad = np.flatnonzero(~valid) + 1          # invalid state indices, 1-based
    if len(bad) == 0:
        return True, s
    j = (bad - 1) % s + 1                      # position inside its stratum
    it = (s - j + 1) if backward else j
    return False, int(it.min())


# ------------------------------------------------------------ nearest neighbours

def nn_distances(points: np.ndarray, q) -> np.ndarray:
    """Distances of q to the (dim, n) float32 SoA points (nn.py:45-51)."""
    qv = np.asarray(q, dtype=F32).reshape(-1)
    diff = np.asarray(points, dtype=F32) - qv[:, None]
    return np.sqrt(np.sum(diff * diff, axis=0, dtype=F32))


def nn_k_nearest(points: np.ndarray, q, k: int) -> tuple[np.ndarray, np.ndarray]:
    """(indices, distances) of the k closest, ascending, ties to the smaller
    index (nn.py:60-69 stable argsort)."""
    d = nn_distances(points, q)
    order = np.argsort(d, kind="stable")[:k]
    return order, d[order]
