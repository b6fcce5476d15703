"""Lower a ``KinematicProgram`` (+ self-collision pairs) to sm_100a CUDA C++.

This is the B200 counterpart of the reference's lane interpreter
(pkg/src/vecmp/program.py:157-214 driving collision.py:293-408): instead of
dispatching one numpy ufunc per op over W lanes, the op list becomes
straight-line register code with one configuration per thread, compiled once
per robot by NVRTC (csrc/vmp.cu) and cached as a cubin.

Generated kernels (all take one by-value argument struct from csrc/vmp_abi.h):

  vmp_fk_rows            every op row (evaluate_program's Scratch)
  vmp_fk_spheres         3 rows per marker (sphere centres; HBM-bound kernel)
  vmp_validate_p{P}_s{S} fused FK + self-collision + environment narrowphase,
                         packed uint32 verdict bitmask (P: coarse prune,
                         S: 0 dense, 1 stop when every lane of the warp is
                         invalid = reference collision.py:403)
  vmp_motion_p{P}_s{S}   warp-per-edge raked motion validation; S=2 stops at
                         the first invalid lane (W multiple of 32), S=1 keeps
                         exact W-block counts for any W

Kernel structure: FK for all spheres first (cheap, ~150
flop), then self pairs with compile-time thresholds, then an obstacle-major
sweep - each obstacle record is read once from shared memory and tested
against every config-dependent fine sphere held in registers.  Spheres whose
centres are program constants (e.g. the arm7 base) are tested against the
environment once per CTA, not once per configuration.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .program import ADD, CONST, COS, FINE, INPUT, MUL, NEG, SIN, SUB

CSRC = Path(__file__).resolve().parent / "csrc"
BLOCK = 128
GROUP_SIZE = 3          # dynamic spheres per broadphase group
SPLIT = 4               # warps per configuration slice in the small-batch validate kernels
SPLITS = (4,)           # split validate kernels emitted (a 2-warp split measured no
                        # faster at 16K-256K configurations, scripts/exp_stream.py)
MOTION_MIN_CTAS = 5     # occupancy target of the register-capped rake variant (6-8: spills, measured slower)
FK_SMEM_TILE = 160 * 1024   # largest vmp_fk_spheres centre tile (shared memory bytes)


def fk_tiling(n_rows: int) -> tuple[int, int]:
    """(configurations per thread, tile buffers) of vmp_fk_spheres.

    Longer contiguous row segments per bulk store write faster (measured,
    scripts/exp_fk_tile.py: 0.83 -> 0.91 of HBM from 1 KB to 2 KB rows for
    arm7), so take the largest 1 / 2 / 4 configurations per thread whose tile
    fits; double-buffer when two tiles fit in 80 KB.  0 buffers: the rows do
    not fit at all and the kernel uses streaming stores only.
    """
    for per in (4, 2, 1):
        tile_bytes = n_rows * BLOCK * per * 4
        if tile_bytes <= FK_SMEM_TILE:
            return per, (2 if 2 * tile_bytes <= 80 * 1024 else 1)
    return 1, 0
CODEGEN_VERSION = 49
# packed FFMA2 (fma.rn.f32x2) broadphase chains; VMP_NO_FFMA2=1 at codegen: scalar
FFMA2 = __import__("os").environ.get("VMP_NO_FFMA2", "") != "1"
# experiment switches (comma-separated names in VMP_EXP at codegen; scripts/exp_*.sh)
EXP = frozenset(x for x in __import__("os").environ.get("VMP_EXP", "").split(",") if x)
# per-item debug timeline records in the rake (scripts/exp_motion_trace.py sets
# this before codegen runs); off in production - they cost ~2 % of the step
TRACE_ITEMS = __import__("os").environ.get("VMP_MOTION_TRACE_ITEMS", "") == "1"


def f32_literal(value: float) -> str:
    """Exact float32 literal (hex float) of ``np.float32(value)``."""
    v = np.float32(value)
    if v == 0:
        return "-0.0f" if np.signbit(v) else "0.0f"
    if not np.isfinite(v):
        raise ValueError(f"non-finite constant {value!r} in program")
    return f"{float(v).hex()}f".replace("0x", "0x")


@dataclass(frozen=True)
class FineSphere:
    slot: int          # index among fine markers (program order)
    link: int
    index: int
    radius: float
    xyz: tuple         # op ids
    const: bool        # centre independent of the configuration


@dataclass(frozen=True)
class RobotLayout:
    """Everything codegen derives from (program, pairs)."""

    dof: int
    n_ops: int
    n_markers: int
    fine: tuple
    coarse: dict       # link -> (radius, xyz) for links with >= 2 fine spheres
    pairs: tuple       # (slot_a, slot_b, thr_f32)
    has_cc: bool       # pairs given -> collision kernels emitted
    link_pairs: frozenset = frozenset()   # checked (lo, hi) link pairs
    home: tuple = (0.0, 0.0, 0.0)         # environment frame origin (robot_home)

    @property
    def dynamic(self) -> list:
        return [s for s in self.fine if not s.const]

    @property
    def const_spheres(self) -> list:
        return [s for s in self.fine if s.const]


def derive_layout(program, pairs=None) -> RobotLayout:
    kinds = np.asarray(program.kinds)
    fine: list[FineSphere] = []
    coarse_of: dict[int, tuple] = {}
    per_link: dict[int, list[int]] = {}
    for m in program.checks:
        xyz = tuple(int(v) for v in m.xyz)
        if m.level == FINE:
            slot = len(fine)
            const = all(int(kinds[v]) == CONST for v in xyz)
            fine.append(FineSphere(slot, int(m.link), int(m.index), float(m.radius), xyz, const))
            per_link.setdefault(int(m.link), []).append(slot)
        else:
            coarse_of[int(m.link)] = (float(m.radius), xyz)
    coarse = {link: coarse_of[link] for link, slots in per_link.items()
              if len(slots) >= 2 and link in coarse_of}
    pair_list = []
    if pairs is not None:
        for lo, hi in sorted(tuple(sorted(p)) for p in pairs.pairs):
            for sb in per_link.get(hi, ()):
                for sa in per_link.get(lo, ()):
                    ra, rb = fine[sa].radius, fine[sb].radius
                    thr = np.float32(np.float32(rb + ra) * np.float32(rb + ra))
                    pair_list.append((sa, sb, float(thr)))
    return RobotLayout(dof=int(program.dof), n_ops=len(kinds), n_markers=len(program.checks),
                       fine=tuple(fine), coarse=coarse, pairs=tuple(pair_list),
                       has_cc=pairs is not None,
                       link_pairs=frozenset(tuple(sorted(p)) for p in pairs.pairs)
                       if pairs is not None else frozenset(),
                       home=robot_home(program))


def _fk_lines(program) -> list[str]:
    """Straight-line float32 FK: one SSA value per op (contraction allowed)."""
    kinds = [int(k) for k in program.kinds]
    a = [int(x) for x in program.a]
    b = [int(x) for x in program.b]
    values = [float(x) for x in program.values]
    cos_of = {a[i]: i for i, k in enumerate(kinds) if k == COS}
    sin_of = {a[i]: i for i, k in enumerate(kinds) if k == SIN}
    done: set[int] = set()
    lines: list[str] = []
    for i, k in enumerate(kinds):
        if i in done:
            continue
        if k == CONST:
            lines.append(f"const float v{i} = {f32_literal(values[i])};")
        elif k == INPUT:
            lines.append(f"const float v{i} = q[{int(values[i])}];")
        elif k == ADD:
            lines.append(f"const float v{i} = v{a[i]} + v{b[i]};")
        elif k == SUB:
            lines.append(f"const float v{i} = v{a[i]} - v{b[i]};")
        elif k == MUL:
            lines.append(f"const float v{i} = v{a[i]} * v{b[i]};")
        elif k == NEG:
            lines.append(f"const float v{i} = -v{a[i]};")
        elif k in (SIN, COS):
            arg = a[i]
            si, ci = sin_of.get(arg), cos_of.get(arg)
            if si is not None and ci is not None:
                lines.append(f"float v{si}, v{ci}; vmp_sincos(v{arg}, &v{si}, &v{ci});")
                done.update((si, ci))
            elif k == SIN:
                lines.append(f"float v{i}, vdummy{i}; vmp_sincos(v{arg}, &v{i}, &vdummy{i});")
            else:
                lines.append(f"float vdummy{i}, v{i}; vmp_sincos(v{arg}, &vdummy{i}, &v{i});")
        else:
            raise ValueError(f"unknown op kind {k} at {i}")
    return lines


def _xyz(s: FineSphere) -> tuple[str, str, str]:
    return tuple(f"v{v}" for v in s.xyz)


def _values_at_zero(program) -> np.ndarray:
    """float64 value of every op at the zero configuration (codegen-time
    analysis only: the home point and the operand choice of ``_HomeShift``)."""
    kinds, a, b, values = program.kinds, program.a, program.b, program.values
    val = np.zeros(len(kinds))
    for i, k in enumerate(int(k) for k in kinds):
        x = val[a[i]] if a[i] >= 0 else 0.0
        y = val[b[i]] if b[i] >= 0 else 0.0
        val[i] = {CONST: values[i], INPUT: 0.0, ADD: x + y, SUB: x - y, MUL: x * y, NEG: -x,
                  SIN: np.sin(x), COS: np.cos(x)}[k]
    return val


HOME_RADIUS = 2.0    # m: robots whose sphere centroid is nearer the origin keep the world frame


def robot_home(program) -> tuple:
    """Origin of the environment frame the collision kernels work in: the mean
    sphere centre at the zero configuration, rounded to 1/64 m (exact in
    float32), or the world origin when that centroid lies within
    ``HOME_RADIUS``.  Obstacle records are packed relative to it (vmp_env_create_at),
    so the expanded test forms (|c|^2 + |o|^2 - 2 c.o) never cancel
    |c|^2-sized terms for a robot far from the world origin."""
    if not program.checks:
        return (0.0, 0.0, 0.0)
    val = _values_at_zero(program)
    c = np.asarray([[val[v] for v in m.xyz] for m in program.checks]).mean(axis=0)
    if np.linalg.norm(c) <= HOME_RADIUS:
        # near the world origin the expanded forms are accurate to < 2e-5 m
        # and the unshifted sums are ~1 % faster in the rake
        return (0.0, 0.0, 0.0)
    return tuple(float(v) for v in np.round(c * 64.0) / 64.0)


class _HomeShift:
    """Sphere-centre coordinates minus the home point, folded into the op DAG.

    shift(op, axis) is an expression for value(op) - home[axis]: a CONST op
    folds to a new literal; ADD / SUB move the subtraction into the operand
    that carries the translation (the one nearer home at the zero
    configuration), so along the usual translation chains no operation is
    added - the rewritten sums replace the originals, which become dead; any
    other op gets one FADD.  Errors stay linear in |home| (one rounding of a
    value near home), unlike the quadratic cancellation of the expanded forms.
    """

    def __init__(self, program, home):
        self.kinds = [int(k) for k in program.kinds]
        self.a = [int(x) for x in program.a]
        self.b = [int(x) for x in program.b]
        self.values = [float(v) for v in program.values]
        self.home = home
        self.val = _values_at_zero(program) if any(home) else None
        self.memo: dict = {}
        self.lines: list[str] = []

    def __call__(self, op: int, axis: int) -> str:
        o = self.home[axis]
        if o == 0.0:
            return f"v{op}"
        key = (op, axis)
        if key in self.memo:
            return self.memo[key]
        k = self.kinds[op]
        if k == CONST:
            expr = f32_literal(self.values[op] - o)
        else:
            if k == ADD:
                x, y = self.a[op], self.b[op]
                if abs(self.val[y] - o) < abs(self.val[x] - o):
                    x, y = y, x
                rhs = f"{self(x, axis)} + v{y}"
            elif k == SUB:
                rhs = f"{self(self.a[op], axis)} - v{self.b[op]}"
            else:
                rhs = f"v{op} - {f32_literal(o)}"
            expr = f"h{len(self.lines)}"
            self.lines.append(f"  const float {expr} = {rhs};")
        self.memo[key] = expr
        return expr

    def xyz(self, ops) -> tuple[str, str, str]:
        return tuple(self(int(v), axis) for axis, v in enumerate(ops))


def _state_function(lay: RobotLayout, program) -> str:
    dyn = lay.dynamic
    out = []
    emit = out.append
    emit("template <int STOP, bool PRUNE, bool TWO = (STOP == 2), bool NO_SPH = false>")
    emit("__device__ __forceinline__ bool vmp_state(const float *q, const float4 *__restrict__ env,")
    emit("                                          int ns, int nc, int nb, bool ok,")
    emit("                                          int sub = 0, int split = 1,")
    emit("                                          unsigned long long *bar = nullptr,")
    emit("                                          bool pairs_rt = true) {")
    emit("  // pairs_rt: the bound-pair records lie behind the obstacle records at env")
    emit("  (void)pairs_rt;")
    emit("  // split > 1: this thread handles obstacles k = sub (mod split) and self")
    emit("  // pairs i = sub (mod split) of its configuration (small-batch kernels)")
    emit("  (void)env; (void)ns; (void)nc; (void)nb;")
    for line in _FK_BODY_PLACEHOLDER:
        emit(line)
    # every collision test runs in the environment frame centred at the robot's
    # home point (obstacle records are packed relative to it): sphere centres
    # minus home, folded into the FK sums (_HomeShift) - no per-state cost
    shift = _HomeShift(program, lay.home)
    env_xyz = {s.slot: shift.xyz(s.xyz) for s in lay.fine}
    coarse_env = {link: shift.xyz(xyz) for link, (_, xyz) in lay.coarse.items()}
    for line in shift.lines:
        emit(line)

    def _exyz(s: FineSphere) -> tuple[str, str, str]:
        return env_xyz[s.slot]
    emit("#define VMP_STOP_NOW ((STOP == 1 && !__any_sync(VMP_FULL, ok)) || "
         "(STOP == 2 && __any_sync(VMP_FULL, !ok && vmp_inr)))")
    emit("  const bool vmp_inr = ok;")
    # all-invalid exits (STOP 1) rarely fire at 20-60 % collision rates: vote every
    # 4th obstacle; any-invalid exits (STOP 2, motion) every 2nd
    emit("  constexpr int VMP_STOP_MASK = STOP == 1 ? 3 : 1;")
    emit("  (void)vmp_inr;")
    fine = lay.fine
    # batch validation (random configurations in a warp): plain self pairs first,
    # before the broadphase state is live; the motion rake (coherent lanes along
    # an edge, STOP 2) culls whole pair buckets with the group bounds below
    emit("  constexpr bool CULL_SELF = STOP == 2;")   # batch mode: culling measured slower (cfg4 413 vs 336 us)
    # per-sphere constants
    for s in dyn:
        x, y, z = _exyz(s)
        rs2 = np.float32(np.float32(s.radius) * np.float32(s.radius))
        emit(f"  const float S{s.slot} = vmp_sphere_S({x}, {y}, {z}, {f32_literal(rs2)});")
    # broadphase groups: consecutive dynamic spheres, bounded per lane by a sphere
    # centred on the group's middle sphere with the exact (inflated) covering
    # radius - one bound test per group per obstacle replaces one per sphere
    n_groups = -(-len(dyn) // GROUP_SIZE)
    # VMP_EXP=evengroups: an odd group count costs as much per obstacle as the
    # next even one (two groups share a packed bound chain), but the tighter
    # split needs more registers: measured slower (arm7 rake 37.0 -> 41.1 us,
    # config 3 158 -> 166 us)
    if FFMA2 and n_groups % 2 == 1 and n_groups < len(dyn) and "evengroups" in EXP:
        n_groups += 1
        cuts = [round(i * len(dyn) / n_groups) for i in range(n_groups + 1)]
        groups = [dyn[cuts[i]:cuts[i + 1]] for i in range(n_groups)]
    else:
        groups = [dyn[i:i + GROUP_SIZE] for i in range(0, len(dyn), GROUP_SIZE)]
    emit("  constexpr bool CULL = STOP != 0;")
    emit(f"  constexpr bool VMP_WARP_VOTE = {'true' if 'warpvote' in EXP else 'false'};")
    emit(f"  constexpr bool VMP_RAKE_VOTE = {'true' if 'rakevote' in EXP else 'false'};")
    main_emit, group_lines = emit, []
    emit = group_lines.append          # group bounds are emitted after the batch self pairs
    for gi, grp in enumerate(groups):
        mid = grp[len(grp) // 2]
        mx, my, mz = _exyz(mid)
        emit(f"  float G{gi}R = {f32_literal(mid.radius)};")
        for s in grp:
            if s is mid:
                continue
            x, y, z = _exyz(s)
            emit(f"  G{gi}R = fmaxf(G{gi}R, vmp_dist({x}, {y}, {z}, {mx}, {my}, {mz}) + "
                 f"{f32_literal(s.radius)});")
        emit(f"  G{gi}R = fmaf(G{gi}R, 1.000002f, 1e-6f);")
        ex, ey, ez = _exyz(mid)
        emit(f"  const float G{gi}S = vmp_sphere_S({ex}, {ey}, {ez}, G{gi}R * G{gi}R);")
        emit(f"  const float G{gi}M = -2.0f * G{gi}R;")
    # broadphase bound tests of two groups per packed FFMA2 chain (bit-identical
    # to the scalar chains); an odd last group stays scalar
    pairs = [(groups[i], i) for i in range(0, len(groups) - 1, 2)] if FFMA2 else []
    for _, gi in pairs:
        a, b = groups[gi], groups[gi + 1]
        (ax, ay, az), (bx, by, bz) = _exyz(a[len(a) // 2]), _exyz(b[len(b) // 2])
        emit(f"  const vmp_f2 Q{gi}X = vmp_pk({ax}, {bx}), Q{gi}Y = vmp_pk({ay}, {by}), "
             f"Q{gi}Z = vmp_pk({az}, {bz});")
        emit(f"  const vmp_f2 Q{gi}S = vmp_pk(G{gi}S, G{gi + 1}S), Q{gi}M = vmp_pk(G{gi}M, G{gi + 1}M);")
    emit = main_emit

    # narrowphase units: two spheres per packed (FFMA2) test.  Only spheres
    # whose three coordinates all depend on the configuration are paired: a constant
    # coordinate (0 along an axis the sphere never leaves, e.g. a torso
    # sphere) lets the compiler fold terms of the scalar form away, which a
    # packed operand would carry as real work.  The rest stay scalar.
    kinds_all = [int(k) for k in program.kinds]

    def fully_dynamic(s):
        return all(kinds_all[v] != CONST for v in s.xyz)
    units: list[tuple] = []            # (sphere,) or (sphere_a, sphere_b)
    if FFMA2 and "nopack" not in EXP:
        # spheres of two adjacent groups pair position by position with the mids
        # aligned: the mids' pair is then also the packed operand of the
        # broadphase chain (one register pair serves both)
        mate: dict[int, FineSphere] = {}
        for gi in range(0, len(groups) - 1, 2):
            a, b = groups[gi], groups[gi + 1]
            ma, mb = len(a) // 2, len(b) // 2
            for d in range(-GROUP_SIZE, GROUP_SIZE + 1):
                if 0 <= ma + d < len(a) and 0 <= mb + d < len(b):
                    sa, sb = a[ma + d], b[mb + d]
                    if fully_dynamic(sa) and fully_dynamic(sb):
                        mate[sa.slot], mate[sb.slot] = sb, sa
        # leftover movers pair up in order
        rest = [s for s in dyn if fully_dynamic(s) and s.slot not in mate]
        for i in range(0, len(rest) - 1, 2):
            mate[rest[i].slot], mate[rest[i + 1].slot] = rest[i + 1], rest[i]
        seen: set = set()
        for s in dyn:
            if s.slot in seen:
                continue
            if s.slot in mate:
                units.append((s, mate[s.slot]))
                seen.update((s.slot, mate[s.slot].slot))
            else:
                units.append((s,))
                seen.add(s.slot)
    else:
        units = [(s,) for s in dyn]
    for ui, u in enumerate(units):
        if len(u) == 2:
            (ax, ay, az), (bx, by, bz) = _exyz(u[0]), _exyz(u[1])
            emit(f"  const vmp_f2 P{ui}X = vmp_pk({ax}, {bx}), P{ui}Y = vmp_pk({ay}, {by}), "
                 f"P{ui}Z = vmp_pk({az}, {bz});")
            emit(f"  const vmp_f2 P{ui}S = vmp_pk(S{u[0].slot}, S{u[1].slot});")

    # batch validation (unrelated configurations in a warp): every self pair, in
    # expanded form |a|^2 + |b|^2 - 2 a.b against thr - ra^2 - rb^2 (S = |c|^2 -
    # rs^2 is shared with the obstacle tests), two partners of one sphere per
    # packed chain when they share a narrowphase unit: 3 issue slots per pair
    # instead of 7 (config 4 carries 267 pairs per configuration).  Before the
    # group bounds are live.  The rake (STOP 2) culls pair buckets instead.
    vals = np.asarray(program.values, dtype=np.float64)

    def rs2_of(sp):
        return np.float32(np.float32(sp.radius) * np.float32(sp.radius))

    def s_expr(sp):
        if not sp.const:
            return f"S{sp.slot}"
        c = np.asarray([np.float32(vals[v] - o) for v, o in zip(sp.xyz, lay.home)], dtype=np.float64)
        return f32_literal(float(c @ c) - float(rs2_of(sp)))

    def t_lit(sa, sb, thr):
        return f32_literal(float(np.float32(thr)) - float(rs2_of(fine[sa])) - float(rs2_of(fine[sb])))
    # the pair relation is symmetric: sphere c broadcasts (-2 c, S_c) and every
    # unit whose two spheres are both partners of c takes one packed test
    thr_of = {frozenset((sa, sb)): thr for sa, sb, thr in lay.pairs}
    nbrs: dict[int, set] = {}
    for sa, sb, _ in lay.pairs:
        nbrs.setdefault(sa, set()).add(sb)
        nbrs.setdefault(sb, set()).add(sa)
    todo = set(thr_of)
    plan: dict[int, list] = {}
    for c in sorted(nbrs, key=lambda c: -len(nbrs[c])):
        for ui, u in enumerate(units):
            if len(u) == 2 and all(frozenset((sp.slot, c)) in todo for sp in u):
                plan.setdefault(c, []).append(("pk", ui))
                todo -= {frozenset((sp.slot, c)) for sp in u}
    for pair in sorted(todo, key=sorted):
        sa, sb = sorted(pair)
        c = sb if sb in plan or sa not in plan else sa
        plan.setdefault(c, []).append(("one", sa if c == sb else sb))
    emit("  if constexpr (!CULL_SELF) {")
    ti = 0
    for c, tests in plan.items():
        bx, by, bz = _exyz(fine[c])
        emit(f"    {{ const float mx = -2.0f * {bx}, my = -2.0f * {by}, mz = -2.0f * {bz}, "
             f"sb = {s_expr(fine[c])};")
        for kind, x in tests:
            if kind == "pk":
                u0, u1 = units[x]
                emit(f"      if (sub == {ti} % split) ok &= vmp_clear_pair2(P{x}X, P{x}Y, P{x}Z, P{x}S, "
                     f"mx, my, mz, sb, {t_lit(u0.slot, c, thr_of[frozenset((u0.slot, c))])}, "
                     f"{t_lit(u1.slot, c, thr_of[frozenset((u1.slot, c))])});")
            else:
                ax, ay, az = _exyz(fine[x])
                emit(f"      if (sub == {ti} % split) ok &= vmp_clear_pair_x({ax}, {ay}, {az}, "
                     f"{s_expr(fine[x])}, mx, my, mz, sb, {t_lit(x, c, thr_of[frozenset((x, c))])});")
            ti += 1
        emit("    }")
    emit("  }")
    for line in group_lines:
        emit(line)

    def bound_masks(ind: str) -> None:
        """Per obstacle: shift every group's near bit into its per-lane mask."""
        paired = set()
        for _, gi in pairs:
            emit(ind + f"{{ const vmp_f2 w = vmp_near2(Q{gi}X, Q{gi}Y, Q{gi}Z, Q{gi}S, Q{gi}M, bnd, brad); "
                 f"n{gi} = vmp_push_sign(n{gi}, vmp_lo(w)); "
                 f"n{gi + 1} = vmp_push_sign(n{gi + 1}, vmp_hi(w)); }}")
            paired.update((gi, gi + 1))
        for gi, grp in enumerate(groups):
            if gi not in paired:
                mx, my, mz = _exyz(grp[len(grp) // 2])
                emit(ind + f"n{gi} = vmp_push_sign(n{gi}, "
                     f"vmp_near1({mx}, {my}, {mz}, G{gi}S, G{gi}M, bnd, brad));")

    def bound_masks_pair(ind: str) -> None:
        """Per TWO obstacles (one bound-pair record: bx2, by2, bz2, bw2, br2): the
        odd group takes both bounds in one packed chain; obstacle 2p + 1 is
        pushed first so that bit j of a mask stays obstacle j of the chunk."""
        paired = set()
        for _, gi in pairs:
            for half in ("hi", "lo"):
                emit(ind + f"{{ const vmp_f2 w = vmp_near2s(Q{gi}X, Q{gi}Y, Q{gi}Z, Q{gi}S, Q{gi}M, "
                     f"vmp_{half}(bx2), vmp_{half}(by2), vmp_{half}(bz2), vmp_{half}(bw2), vmp_{half}(br2)); "
                     f"n{gi} = vmp_push_sign(n{gi}, vmp_lo(w)); "
                     f"n{gi + 1} = vmp_push_sign(n{gi + 1}, vmp_hi(w)); }}")
            paired.update((gi, gi + 1))
        for gi, grp in enumerate(groups):
            if gi not in paired:
                mx, my, mz = _exyz(grp[len(grp) // 2])
                emit(ind + f"{{ const vmp_f2 w = vmp_near1x2({mx}, {my}, {mz}, G{gi}S, G{gi}M, "
                     f"bx2, by2, bz2, bw2, br2); "
                     f"n{gi} = vmp_push_sign(vmp_push_sign(n{gi}, vmp_hi(w)), vmp_lo(w)); }}")

    # the rake tests two obstacle bounds per packed chain for the odd group
    # (bound-pair records, csrc/vmp_abi.h VMP_PAIR_F4): 26 instead of 34
    # instructions per two obstacles on arm7
    use_pairs = FFMA2 and len(groups) % 2 == 1 and "nopairs" not in EXP

    def bound_terms() -> list[str]:
        """Per obstacle: the expanded bound distance of every group, as terms
        whose minimum decides "near" (packed pairs first)."""
        terms = [f"vmp_sphere_w2(Q{gi}X, Q{gi}Y, Q{gi}Z, Q{gi}S, Q{gi}M, bnd, brad)" for _, gi in pairs]
        paired = {gi for _, gi in pairs} | {gi + 1 for _, gi in pairs}
        for gi, grp in enumerate(groups):
            if gi not in paired:
                mx, my, mz = _exyz(grp[len(grp) // 2])
                terms.append(f"vmp_sphere_w({mx}, {my}, {mz}, G{gi}S, G{gi}M, bnd, brad)")
        return terms
    # self-collision pairs (compile-time thresholds), bucketed by group pair;
    # constant spheres are singleton groups with their exact centre and radius.
    # A bucket is skipped when no lane has its two group bounds overlapping.
    # Buckets of two groups holding spheres of joint-adjacent links (a link
    # pair with spheres on both links that is not checked) are near in
    # practically every warp (measured on config 2), so their pairs are tested
    # without the bucket test.
    group_of: dict[int, tuple] = {}
    links_of: dict[str, set] = {}
    for gi, grp in enumerate(groups):
        mxyz = _exyz(grp[len(grp) // 2])
        for s in grp:
            group_of[s.slot] = (f"g{gi:03d}", mxyz, f"G{gi}R")
            links_of.setdefault(f"g{gi:03d}", set()).add(s.link)
    for s in lay.const_spheres:
        group_of[s.slot] = (f"c{s.slot:03d}", _exyz(s), f32_literal(s.radius))
        links_of.setdefault(f"c{s.slot:03d}", set()).add(s.link)

    def touching(ka, kb):
        return any(la != lb and (min(la, lb), max(la, lb)) not in lay.link_pairs
                   for la in links_of[ka] for lb in links_of[kb])
    buckets: dict[tuple, list] = {}
    for sa, sb, thr in lay.pairs:
        ka, kb = group_of[sa][0], group_of[sb][0]
        key = (ka, kb) if ka <= kb else (kb, ka)
        buckets.setdefault(key, []).append((sa, sb, thr))
    by_name = {v[0]: v for v in group_of.values()}
    emit("  if constexpr (CULL_SELF) {")
    for (ka, kb), items in buckets.items():
        tests = []
        for sa, sb, thr in items:
            ax, ay, az = _exyz(fine[sa])
            bx, by, bz = _exyz(fine[sb])
            tests.append(f"ok &= vmp_clear_pair({bx}, {by}, {bz}, {ax}, {ay}, {az}, "
                         f"{f32_literal(thr)}); ")
        if ka == kb or (ka[0] == "c" and kb[0] == "c") or touching(ka, kb):
            for t in tests:
                emit("  " + t)
            continue
        (_, (ax, ay, az), ra), (_, (bx, by, bz), rb) = by_name[ka], by_name[kb]
        emit(f"  if (__any_sync(VMP_FULL, !vmp_clear_pair({ax}, {ay}, {az}, {bx}, {by}, "
             f"{bz}, ({ra} + {rb}) * ({ra} + {rb})))) {{")
        for t in tests:
            emit("    " + t)
        emit("  }")
    emit("  }")
    emit("  if (VMP_STOP_NOW) return ok;")
    coarse_links = {link for link in lay.coarse}
    by_link: dict[int, list[FineSphere]] = {}
    for s in dyn:
        by_link.setdefault(s.link, []).append(s)

    def pruned(s):
        return s.link in coarse_links and len(by_link[s.link]) >= 2
    # per-link coarse prune (reference collision.py:367-381): in dense mode only,
    # unless VMP_EXP=coarse - the group broadphase already culls per 3 spheres
    prune_expr = "PRUNE" if "coarse" in EXP else "(PRUNE && !CULL)"
    pruned_links = sorted({s.link for u in units if all(pruned(x) for x in u) for s in u})

    def group_tests(test_fn, coarse_fn, ind: str = "    ") -> None:
        """Every narrowphase unit against the obstacle record in r0..r3.  A
        unit whose spheres all sit on links with a coarse sphere (>= 2 fine
        spheres) is skipped when every lane's coarse spheres are clear; each
        link's coarse vote is taken once per obstacle."""
        for link in pruned_links:
            emit(ind + f"const bool near{link} = !{prune_expr} || "
                 f"__any_sync(VMP_FULL, !{coarse_fn(link)});")
        for ui, u in enumerate(units):
            test = test_fn(u[0]) if len(u) == 1 else test_fn(u[0], u[1], ui)
            if all(pruned(s) for s in u):
                cond = " || ".join(f"near{link}" for link in sorted({s.link for s in u}))
                emit(ind + f"if ({cond}) ok &= {test};")
            else:
                emit(ind + f"ok &= {test};")

    def coarse_xyz(link):
        return lay.coarse[link][0], coarse_env[link]

    def sph_test(s, s2=None, ui=None):
        if s2 is not None:
            return (f"vmp_clear_sphere2(P{ui}X, P{ui}Y, P{ui}Z, P{ui}S, {f32_literal(2.0 * np.float32(s.radius))}, "
                    f"{f32_literal(2.0 * np.float32(s2.radius))}, r0, r1.x)")
        x, y, z = _exyz(s)
        return f"vmp_clear_sphere({x}, {y}, {z}, S{s.slot}, {f32_literal(-2.0 * np.float32(s.radius))}, r0, r1.x)"

    def sph_coarse(link):
        r, (x, y, z) = coarse_xyz(link)
        rs2 = np.float32(np.float32(r) * np.float32(r))
        return (f"vmp_clear_sphere({x}, {y}, {z}, vmp_sphere_S({x}, {y}, {z}, {f32_literal(rs2)}), "
                f"{f32_literal(-2.0 * np.float32(r))}, r0, r1.x)")

    def cap_test(s, s2=None, ui=None):
        if s2 is not None:
            return (f"vmp_clear_capsule2(P{ui}X, P{ui}Y, P{ui}Z, P{ui}S, {f32_literal(2.0 * np.float32(s.radius))}, "
                    f"{f32_literal(2.0 * np.float32(s2.radius))}, r0, r1, r2)")
        x, y, z = _exyz(s)
        return f"vmp_clear_capsule({x}, {y}, {z}, S{s.slot}, {f32_literal(-2.0 * np.float32(s.radius))}, r0, r1, r2)"

    def cap_coarse(link):
        r, (x, y, z) = coarse_xyz(link)
        rs2 = np.float32(np.float32(r) * np.float32(r))
        return (f"vmp_clear_capsule({x}, {y}, {z}, vmp_sphere_S({x}, {y}, {z}, {f32_literal(rs2)}), "
                f"{f32_literal(-2.0 * np.float32(r))}, r0, r1, r2)")

    def box_fn(radius):
        return "vmp_clear_box_small" if radius < 1.0 else "vmp_clear_box_any"

    def box_test(s, s2=None, ui=None):
        if s2 is not None:
            ra2 = np.float32(np.float32(s.radius) * np.float32(s.radius))
            rb2 = np.float32(np.float32(s2.radius) * np.float32(s2.radius))
            small = lambda r: "true" if r < 1.0 else "false"
            return (f"vmp_clear_box2<{small(s.radius)}, {small(s2.radius)}>(P{ui}X, P{ui}Y, P{ui}Z, "
                    f"{f32_literal(ra2)}, {f32_literal(rb2)}, r0, r1, r2, r3)")
        x, y, z = _exyz(s)
        rs2 = np.float32(np.float32(s.radius) * np.float32(s.radius))
        return f"{box_fn(s.radius)}({x}, {y}, {z}, {f32_literal(rs2)}, r0, r1, r2, r3)"

    def box_coarse(link):
        r, (x, y, z) = coarse_xyz(link)
        rs2 = np.float32(np.float32(r) * np.float32(r))
        return f"{box_fn(r)}({x}, {y}, {z}, {f32_literal(rs2)}, r0, r1, r2, r3)"

    def kind_loop(count: str, f4: str, base: str, loads: str, bound: str, radius: str, test_fn,
                  coarse_fn, pair_base: str = ""):
        # dense mode (STOP 0): every obstacle, every test - the honest roofline run
        emit(f"  p = {base} + sub * {f4};")
        emit("  if constexpr (!CULL) {")
        emit(f"    for (int k = sub; k < {count}; k += split, p += split * {f4}) {{")
        emit(f"      const float4 {loads};")
        group_tests(test_fn, coarse_fn, "      ")
        emit("    }")
        emit("  } else if constexpr (TWO ? !VMP_RAKE_VOTE : !VMP_WARP_VOTE) {")
        # batch validation (unrelated configurations in a warp): per-lane near
        # lists.  Pass 1 tests every group bound against every obstacle bound
        # of a 32-obstacle chunk into one bit mask per group per lane; pass 2
        # walks the groups and each lane pops ITS OWN near obstacles, testing
        # only that group's spheres (per-lane record address).  A warp vote
        # here would call an obstacle near when any of 32 unrelated
        # configurations is (35-50 % of obstacles on configs 1 / 3 / 4) and
        # make every lane test every sphere; the lists cut the sphere tests
        # 4-8x (scripts/exp_lane_cull_model.py).  A lane whose verdict is
        # already false drops its lists.
        emit(f"    for (int k0 = sub; k0 < {count}; k0 += 32 * split, p += 32 * split * {f4}) {{")
        emit(f"      const int kn = min(32, ({count} - k0 + split - 1) / split);")
        emit("      unsigned " + ", ".join(f"n{gi} = 0" for gi in range(len(groups))) + ";")
        if use_pairs:
            # rake / unsplit batch kernels with staged pairs: the chunk's bound pairs, last first
            emit("      if ((TWO || split == 1) && pairs_rt) {")
            emit("        const int np = (kn + 1) >> 1;")
            emit(f"        const ulonglong2 *pq = (const ulonglong2 *)({pair_base}) + "
                 f"VMP_PAIR_F4 * ((k0 >> 1) + np - 1);")
            emit("#pragma unroll 1")
            emit("        for (int j = np - 1; j >= 0; --j, pq -= VMP_PAIR_F4) {")
            emit("          const ulonglong2 q0 = pq[0], q1 = pq[1];")
            emit("          const vmp_f2 bx2 = q0.x, by2 = q0.y, bz2 = q1.x, bw2 = q1.y, "
                 "br2 = *(const vmp_f2 *)(pq + 2);")
            bound_masks_pair("          ")
            emit("        }")
            emit("        // an odd chunk: the pad bound was pushed as obstacle kn, never near")
            emit("      } else {")
        emit(f"      const float4 *pp = p + (kn - 1) * split * {f4};")
        emit("#pragma unroll 2")
        emit(f"      for (int j = kn - 1; j >= 0; --j, pp -= split * {f4}) {{")
        emit(f"        const float4 bnd = pp[{bound}];")
        emit(f"        const float brad = {radius};")
        bound_masks("        ")
        emit("      }")
        if use_pairs:
            emit("      }")
        for gi, grp in enumerate(groups):
            emit(f"      while (n{gi} != 0 && ok) {{")
            emit(f"        const int j = __ffs(n{gi}) - 1;")
            emit(f"        n{gi} &= n{gi} - 1;")
            emit(f"        const float4 *pq = p + j * split * {f4};")
            emit(f"        const float4 {loads.replace('p[', 'pq[')};")
            for sph in grp:
                emit(f"        ok &= {test_fn(sph)};")
            emit("      }")
            # the rake stops at the first invalid state of the chunk
            emit("      if (STOP == 2 && VMP_STOP_NOW) return ok;")
        emit("      if (STOP == 1 && VMP_STOP_NOW) return ok;")
        emit("    }")
        emit("  } else if constexpr (STOP == 1 && !TWO) {")
        # warp-vote variant (VMP_EXP=warpvote): one pass, a vote per obstacle
        emit(f"    for (int k = sub; k < {count}; k += split, p += split * {f4}) {{")
        emit(f"      const float4 {loads};")
        # near iff the minimum over the groups of the expanded bound distance
        # is <= the threshold: one compare per obstacle
        emit(f"      const float4 bnd = p[{bound}];")
        emit(f"      const float brad = {radius.replace('pp[', 'p[')};")
        for ti, w in enumerate(bound_terms()):
            emit(f"      float wm0 = {w};" if ti == 0 else f"      wm0 = fminf(wm0, {w});")
        emit("      if (__any_sync(VMP_FULL, wm0 <= bnd.w)) {")
        group_tests(test_fn, coarse_fn, "        ")
        emit("      }")
        emit("      if ((k & VMP_STOP_MASK) == VMP_STOP_MASK && VMP_STOP_NOW) return ok;")
        emit("    }")
        emit("  } else {")
        # motion rake and latency-bound small batches (TWO), two passes per 32
        # obstacles: (1) branch-free bound tests of every group against every
        # obstacle bound into a per-lane bit mask, (2) one warp OR, then full
        # tests only for obstacles near some lane.  Exact: an obstacle lies
        # inside its bound, every sphere inside its group bound.  With split > 1
        # this thread's obstacles are k = sub (mod split).
        emit(f"    for (int k0 = sub; k0 < {count}; k0 += 32 * split, p += 32 * split * {f4}) {{")
        emit(f"      const int kn = min(32, ({count} - k0 + split - 1) / split);")
        emit("      unsigned near = 0;")
        # last obstacle first, the mask shifted up one bit per obstacle: a
        # pointer step and a shift-or per obstacle, no per-j index arithmetic
        emit(f"      const float4 *pp = p + (kn - 1) * split * {f4};")
        emit("#pragma unroll 4")
        emit(f"      for (int j = kn - 1; j >= 0; --j, pp -= split * {f4}) {{")
        emit(f"        const float4 bnd = pp[{bound}];")
        emit(f"        const float brad = {radius};")
        # one compare per obstacle: the minimum over the groups of the expanded
        # bound distance (near iff some group's is <= the threshold)
        for ti, w in enumerate(bound_terms()):
            emit(f"        float wm0 = {w};" if ti == 0 else f"        wm0 = fminf(wm0, {w});")
        emit("        near = (near << 1) | (unsigned)(wm0 <= bnd.w);" if groups else "")
        emit("      }")
        emit("      unsigned todo = __reduce_or_sync(VMP_FULL, near);")
        emit("      while (todo) {")
        emit("        const int j = __ffs(todo) - 1;")
        emit("        todo &= todo - 1;")
        emit(f"        const float4 *pp = p + j * split * {f4};")
        emit(f"        const float4 {loads.replace('p[', 'pp[')};")
        group_tests(test_fn, coarse_fn, "        ")
        emit("        if (VMP_STOP_NOW) return ok;")
        emit("      }")
        emit("    }")
        emit("  }")

    if dyn:
        # the environment copy (cp.async.bulk) was in flight during FK and self pairs
        emit("  if (bar) vmp_mbar_wait(bar, 0);")
        emit("  const float4 *p = env;")
        # NO_SPH: the rake variant for scenes without sphere obstacles carries no
        # sphere code (a smaller hot loop for the instruction cache)
        emit("  if constexpr (!NO_SPH) {")
        pairs0 = "(env + VMP_SPH_F4 * ns + VMP_CAP_F4 * nc + VMP_BOX_F4 * nb)"
        kind_loop("ns", "VMP_SPH_F4", "env", "r0 = p[0], r1 = p[1]", "0", "pp[1].x",
                  sph_test, sph_coarse, pairs0)
        emit("  }")
        kind_loop("nc", "VMP_CAP_F4", "(env + VMP_SPH_F4 * ns)", "r0 = p[0], r1 = p[1], r2 = p[2]",
                  "3", "pp[2].w", cap_test, cap_coarse,
                  f"({pairs0} + VMP_PAIR_F4 * ((ns + 1) >> 1))")
        kind_loop("nb", "VMP_BOX_F4", "(env + VMP_SPH_F4 * ns + VMP_CAP_F4 * nc)",
                  "r0 = p[0], r1 = p[1], r2 = p[2], r3 = p[3]", "4", "pp[3].w",
                  box_test, box_coarse,
                  f"({pairs0} + VMP_PAIR_F4 * (((ns + 1) >> 1) + ((nc + 1) >> 1)))")
    emit("#undef VMP_STOP_NOW")
    emit("  return ok;")
    emit("}")
    return "\n".join(out)


_FK_BODY_PLACEHOLDER = ["  VMP_FK_BODY"]


def _const_check(lay: RobotLayout) -> str:
    """Per-CTA test of configuration-independent spheres against the env."""
    consts = lay.const_spheres
    lines = ["// tid of nth cooperating threads (the CTA, or one warp of the rake)",
             "__device__ __forceinline__ bool vmp_const_clear(const float4 *env, int ns, int nc, int nb,",
             "                                                int tid, int nth) {",
             "  (void)env; (void)ns; (void)nc; (void)nb; (void)tid; (void)nth;",
             "  bool ok = true;"]
    if consts:
        # (const sphere, obstacle) pairs spread over the cooperating threads
        lines.append("  const int nobst = ns + nc + nb;")
        lines.append(f"  for (int t = tid; t < {len(consts)} * nobst; t += nth) {{")
        lines.append("    const int k = t % nobst;")
        lines.append("    switch (t / nobst) {")
        for k, s in enumerate(consts):
            # centre coordinates of a const sphere are CONST ops: exact float32 literals
            lines.append(f"    case {k}: ok &= vmp_sphere_clear_obstacle(env, ns, nc, nb, k, "
                         f"VMP_C{s.slot}X, VMP_C{s.slot}Y, VMP_C{s.slot}Z, {f32_literal(s.radius)}); break;")
        lines.append("    default: break;")
        lines.append("    }")
        lines.append("  }")
    lines.append("  return ok;")
    lines.append("}")
    return "\n".join(lines)


_TRACE_BLOCK = """    if (trace && lane == 0 && t < VMP_TRACE_ITEMS) {   // per item: start, end, round | edge, warp | top
      unsigned long long *rec = a.trace + VMP_TRACE_ITEM0 + 4 * t;
      rec[0] = t_start;
      rec[1] = vmp_gtime();
      rec[2] = ((unsigned long long)ci << 32) | (unsigned long long)ei;
      rec[3] = ((unsigned long long)wid << 48) | (t_top & 0xffffffffffffull);
    }"""


def _kernels(lay: RobotLayout, program) -> str:
    dofp = max(1, lay.dof)
    ld_q = "\n".join(f"    q[{j}] = __ldg(a.q + {j} * a.ld + ii);" for j in range(lay.dof))
    rows = "\n".join(f"    o[{i} * a.ldo] = v{i};" for i in range(lay.n_ops))
    centre_rows = []
    for m, marker in enumerate(program.checks):
        for c, v in enumerate(marker.xyz):
            centre_rows.append(f"    __stcs(o + {3 * m + c} * a.ldo, v{int(v)});")
    centre_rows = "\n".join(centre_rows)
    n_rows = 3 * len(program.checks)
    # two tile buffers when they fit in 80 KB (>= 2 CTAs per SM), else one; the
    # host's fk_tile_bytes (csrc/vmp.cu) applies the same rule
    per, nbuf = fk_tiling(n_rows)
    tile = BLOCK * per
    smem_rows = "\n".join(f"        s[{3 * m + c} * {tile} + c] = v{int(v)};"
                           for m, marker in enumerate(program.checks)
                           for c, v in enumerate(marker.xyz))
    src = f"""
extern "C" __global__ void __launch_bounds__({BLOCK}) vmp_fk_rows(VmpFkArgs a) {{
  for (long long i = blockIdx.x * (long long){BLOCK} + threadIdx.x; i < a.n;
       i += (long long)gridDim.x * {BLOCK}) {{
    const long long ii = i;
    float q[{dofp}];
{ld_q}
    VMP_FK_BODY
    float *o = a.out + i;
{rows}
  }}
}}

// shared memory vmp_fk_spheres needs (read by the host after loading the module)
extern "C" __device__ const int vmp_fk_smem_bytes = {max(nbuf, 1) * n_rows * tile * 4 if nbuf else 0};

extern "C" __global__ void __launch_bounds__({BLOCK}) vmp_fk_spheres(VmpFkArgs a) {{
  // HBM-bound (write side): a CTA computes the centres of a {tile}-configuration
  // tile ({per} per thread, all joints loaded up front) into shared
  // memory ({n_rows} rows x {tile} floats, {nbuf} buffer(s)) and each row leaves as
  // ONE contiguous {tile * 4} B cp.async.bulk (TMA) store that overlaps the next
  // tile's FK.  Unaligned outputs and the partial last tile use streaming stores.
  extern __shared__ float vmp_rows[];                  // [{max(nbuf, 1)}][{n_rows}][{tile}]
  const bool bulk = {"true" if nbuf else "false"} && (a.ldo & 3) == 0 &&
                    ((unsigned long long)a.out & 15) == 0;
  const long long ntiles = (a.n + {tile} - 1) / {tile};
  int buf = 0;
  float qn[{per}][{dofp}];               // next tile's joints, prefetched
  if (blockIdx.x < ntiles) {{
#pragma unroll
    for (int r = 0; r < {per}; ++r) {{
      const long long ii = min((long long)blockIdx.x * {tile} + r * {BLOCK} + threadIdx.x, a.n - 1);
      float *q = qn[r];
{ld_q}
    }}
  }}
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf = (buf + 1) % {max(nbuf, 1)}) {{
    const long long base = tile * {tile};
    const bool full = bulk && base + {tile} <= a.n;    // CTA-uniform
    float *s = vmp_rows + buf * {n_rows * tile};
    float qa[{per}][{dofp}];
#pragma unroll
    for (int r = 0; r < {per}; ++r)
#pragma unroll
      for (int j = 0; j < {dofp}; ++j) qa[r][j] = qn[r][j];
    if (tile + gridDim.x < ntiles) {{
#pragma unroll
      for (int r = 0; r < {per}; ++r) {{
        const long long ii = min((tile + gridDim.x) * {tile} + r * {BLOCK} + threadIdx.x, a.n - 1);
        float *q = qn[r];
{ld_q}
      }}
    }}
    if (full) {{
      vmp_bulk_wait_read<{max(nbuf, 1) - 1}>();   // earlier stores from this buffer have read it
      __syncthreads();
    }}
#pragma unroll
    for (int r = 0; r < {per}; ++r) {{
      const float *q = qa[r];
      const long long i = base + r * {BLOCK} + threadIdx.x;
      VMP_FK_BODY
      if (full) {{
        const int c = r * {BLOCK} + threadIdx.x;
{smem_rows}
      }} else if (i < a.n) {{
        float *o = a.out + i;
{centre_rows}
      }}
    }}
    if (full) {{
      vmp_fence_proxy_async();
      __syncthreads();
      for (int r = threadIdx.x; r < {n_rows}; r += {BLOCK})
        vmp_bulk_s2g(a.out + r * a.ldo + base, s + r * {tile}, {tile * 4});
      vmp_bulk_commit();
    }}
  }}
  vmp_bulk_wait<0>();
}}
"""
    if not lay.has_cc:
        return src
    src += f"""
template <int PRUNE, int STOP, bool STAGED, int SPLIT, bool TWO = false, int NT = {BLOCK}>
__device__ __forceinline__ void vmp_validate_body(const VmpValidateArgs &a) {{
  // NT threads per CTA: {BLOCK}, or 256 for environments whose staged copy
  // limits the CTAs per SM (more warps per copy)
  // SPLIT warps share one 32-configuration slice; warp w tests obstacles and
  // self pairs w (mod SPLIT) and the partial verdict words are AND-ed in smem
  // (more warps and a shorter critical path for latency-bound small batches)
  extern __shared__ float4 vmp_smem[];
  __shared__ unsigned long long vmp_bar;
  __shared__ unsigned vmp_part[NT / 32];
  // a following batch launched with VMP_PDL may start as soon as this grid's
  // CTAs are resident (its inputs are its own; nothing here is waited for)
  asm volatile("griddepcontrol.launch_dependents;");
  // the environment copy overlaps the joint loads, FK and self pairs of the
  // first tile; vmp_state waits for it before the first obstacle
  const float4 *env = STAGED ? vmp_smem : a.env.rec;
  const bool vpairs = STAGED && a.stage == 2;   // bound pairs staged behind the records
  if (STAGED) {{
    vmp_env_begin(a.env, 1, vmp_smem, &vmp_bar, vpairs);
    __syncthreads();
  }}
  bool cclear = true, cdone = false;
  constexpr int TILE = NT / SPLIT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sub = warp % SPLIT;
  const long long stride = (long long)gridDim.x * TILE;
  for (long long base = blockIdx.x * (long long)TILE; base < a.n; base += stride) {{
    const long long i = base + (warp / SPLIT) * 32 + lane;
    const bool inr = i < a.n;
    const long long ii = inr ? i : a.n - 1;
    float q[{dofp}];
{ld_q}
    bool ok = vmp_state<STOP, PRUNE != 0, TWO>(q, env, a.env.ns, a.env.nc, a.env.nb, inr, sub,
                                               SPLIT, STAGED ? &vmp_bar : nullptr, vpairs);
    if (!cdone) {{                            // CTA-uniform: once, after the first tile
      if (STAGED) vmp_mbar_wait(&vmp_bar, 0);
      cclear = __syncthreads_and(vmp_const_clear(env, a.env.ns, a.env.nc, a.env.nb,
                                                   threadIdx.x, blockDim.x));
      cdone = true;
    }}
    ok = ok && cclear;
    const unsigned m = __ballot_sync(VMP_FULL, ok);
    if constexpr (SPLIT == 1) {{
      if (lane == 0 && inr) a.bits[i >> 5] = m;
    }} else {{
      if (lane == 0) vmp_part[warp] = m;
      __syncthreads();
      if (sub == 0 && lane == 0 && inr) {{
        unsigned word = m;
#pragma unroll
        for (int s = 1; s < SPLIT; ++s) word &= vmp_part[warp + s];
        a.bits[i >> 5] = word;
      }}
      __syncthreads();
    }}
  }}
  if (STAGED && !cdone) vmp_mbar_wait(&vmp_bar, 0);   // no tile: still retire the copy
}}

template <int PRUNE, int STOP, bool STAGED, bool NO_SPH = false>
__device__ __forceinline__ void vmp_motion_body(const VmpMotionArgs &a) {{
  // Dynamic-queue rake (csrc/vmp_abi.h).  Round 0 - the first chunk of every
  // edge, discretised by the item itself - is dealt out statically (warp w
  // takes edges w, w + warps, ...): no atomics, nothing to wait for.  An edge
  // whose first iteration passed publishes its remaining chunks as slot
  // records; afterwards warps pop slots until the queue is drained.  Failed
  // edges never enter the queue, nothing is planned or sorted.  Per queue item:
  // one atomic (the next one issued before the current chunk is evaluated), one
  // L2 round trip for the slot (its two words carry the call's tag: valid as
  // soon as they read back), one for the edge rows and the failure record.
  extern __shared__ float4 vmp_smem[];
  __shared__ unsigned long long vmp_bar;
  unsigned long long *trace = a.trace ? a.trace + 8 * blockIdx.x : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = vmp_gtime();
  asm volatile("griddepcontrol.launch_dependents;");
  const float4 *env = a.env.rec;
  if (STAGED) {{
    vmp_env_begin(a.env, 1, vmp_smem, &vmp_bar, true);   // obstacle records + bound pairs
    __syncthreads();                         // the mbarrier is initialised
    env = vmp_smem;
  }}
  bool cclear = true, cdone = false;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long E = a.n_edges, cap = a.slot_cap;
  const unsigned Wu = (unsigned)a.width;
  unsigned long long *const state = a.dq + VMP_DQ_STATE;
  constexpr unsigned long long M40 = (1ull << 40) - 1;
  constexpr int VMP_DQ_KEEP = {next((int(x[4:]) for x in EXP if x.startswith("keep")), 0)};
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const int wid = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  (void)warp;
  // vmp_k_motion_begin resets the queue words, zeroes fail[] and sets the call
  // count: waited for (programmatic dependent launch) before the first write
  // to any of them, i.e. after the first round-0 chunk has been evaluated
  unsigned long long tag = 0;                // 0: the begin kernel has not been waited for
  unsigned taken = 0;
  unsigned long long grab = 0;
  bool have = false;
  long long r0 = wid;                        // next round-0 edge of this warp
  int stripe = wid % VMP_QSTRIPES, dry = 0;
  // chunks [loc_c, loc_end) of edge loc_e that did not fit into the slot array
  // are finished by the warp that owns the edge's round-0 item
  long long loc_e = 0;
  int loc_c = 0, loc_end = 0, loc_n = 0;
  for (;;) {{
{"    const unsigned long long t_top = trace ? vmp_gtime() : 0;" if TRACE_ITEMS else ""}
    long long ei, t = -1;
    int n, ci, fe = 0;
    bool round0 = false;
    if (loc_c < loc_end) {{
      ei = loc_e;
      ci = loc_c++;
      n = loc_n;
      // more than the kept chunk(s): a long overflow run, worth the failure check
      if (loc_end - loc_c > VMP_DQ_KEEP) fe = __ldcg(a.fail + ei);
    }} else if (r0 < E) {{                     // round 0: edge r0, discretised here
      ei = t = r0;
      r0 += nwarps;
      ci = 0;
      round0 = true;
      n = vmp_discretize_edge<{lay.dof}>(a.starts + ei * a.sld, a.goals + ei * a.sld, a.resolution);
    }} else {{
      if (tag == 0) {{
        asm volatile("griddepcontrol.wait;" ::: "memory");
        tag = (1ull + __ldcg(a.dq + VMP_DQ_CALLS) % 65535ull) << 48;
      }}
      // the queue is striped over VMP_QSTRIPES pop counters (slot i belongs to
      // stripe i % VMP_QSTRIPES): thousands of warps leave round 0 within a few
      // microseconds and same-address atomics serialise in L2
      long long i;
      unsigned long long w0, w1, st;
      for (;;) {{
        if (!have && lane == 0) grab = atomicAdd(&a.hdr->counter[16 * stripe], 1ull);
        i = (long long)__shfl_sync(VMP_FULL, grab, 0) * VMP_QSTRIPES + stripe;
        have = false;
        if (i < cap) {{                      // published already (the usual case): no state read
          const ulonglong2 w = __ldca((const ulonglong2 *)(a.slots + 2 * i));
          w0 = w.x;
          w1 = w.y;
          if ((w0 >> 48 << 48) == tag && (w1 >> 48 << 48) == tag) break;
        }}
        unsigned spins = 0;
        unsigned long long spin_t0 = 0;
        for (;;) {{
          ulonglong2 w = make_ulonglong2(0ull, 0ull);
          if (i < cap) w = __ldcg((const ulonglong2 *)(a.slots + 2 * i));
          st = __ldcg(state);
          w0 = w.x;
          w1 = w.y;
          if ((w0 >> 48 << 48) == tag && (w1 >> 48 << 48) == tag) break;
          // not published (yet): more can only come while round 0 is running
          w0 = 0;
          if ((long long)(st >> 40) == E && i >= min((long long)(st & M40), cap)) break;
          // cannot happen (every reserved slot is written by a running warp): fail
          // loudly after 20 s rather than hang the device
          if ((++spins & 1023u) == 0u) {{
            if (spin_t0 == 0) spin_t0 = vmp_gtime();
            else if (vmp_gtime() - spin_t0 > 20000000000ull) __trap();
          }}
          __nanosleep(40);
        }}
        if (w0 != 0) break;
        // this stripe is dry (round 0 is over, so the slot count is final): any other?
        const long long total = min((long long)(st & M40), cap);
        const unsigned long long seen = lane < VMP_QSTRIPES ? __ldcg(&a.hdr->counter[16 * lane]) : 0;
        const unsigned open = __ballot_sync(VMP_FULL, lane < VMP_QSTRIPES &&
                                            (long long)seen * VMP_QSTRIPES + lane < total);
        if (!open || ++dry > 4 * VMP_QSTRIPES) break;
        stripe = __ffs(open) - 1;
      }}
      if (w0 == 0) break;                    // queue drained: this warp is done
      t = E + i;
      // the next pop is in flight while this chunk is evaluated (stopping the
      // prefetch near the end of the queue measured no faster)
      if (lane == 0) grab = atomicAdd(&a.hdr->counter[16 * stripe], 1ull);
      have = true;
      ei = (long long)(w0 & 0x7fffffffull);
      n = (int)(w1 & 0x7fffffffull);
      ci = (int)(((w0 >> 31) & 0x1ffffull) | (((w1 >> 31) & 0x3ffull) << 17));
      fe = __ldcg(a.fail + ei);
    }}
    ++taken;
    const unsigned first_iter = Wu == 32 ? (unsigned)ci + 1 : (32u * (unsigned)ci) / Wu + 1;
{"    const unsigned long long t_start = trace ? vmp_gtime() : 0;" if TRACE_ITEMS else ""}
    if (fe == 0 || 0x7fffffff - fe > (int)first_iter) {{   // else: cannot lower the count
      float s[{dofp}], g[{dofp}];
#pragma unroll
      for (int j = 0; j < {lay.dof}; ++j) {{
        s[j] = __ldg(a.starts + ei * a.sld + j);
        g[j] = __ldg(a.goals + ei * a.sld + j);
      }}
      const unsigned S = Wu == 32 ? ((unsigned)n + 31u) >> 5 : vmp_ceil_div((unsigned)n, Wu);
      const unsigned p = 32u * (unsigned)ci + lane;
      const unsigned j = Wu == 32 ? (unsigned)ci + 1 : p / Wu + 1;
      const unsigned k = Wu == 32 ? (unsigned)lane : p - (j - 1) * Wu;
      const long long idx = (long long)k * S + (a.backward ? (S - j + 1) : j);
      const bool inr = (unsigned long long)p < (unsigned long long)S * Wu && idx <= n;
      const float tt = vmp_rake_param(inr ? idx : 1, n);
      float q[{dofp}];
#pragma unroll
      for (int jj = 0; jj < {lay.dof}; ++jj) q[jj] = vmp_lerp_exact(s[jj], g[jj], tt);
      bool ok = vmp_state<STOP, PRUNE != 0, STOP == 2, NO_SPH>(q, env, a.env.ns, a.env.nc, a.env.nb,
                                                            inr && cclear, 0, 1,
                                                            STAGED ? &vmp_bar : nullptr);
      if (!cdone) {{                         // warp-uniform: once, after the first item
        if (STAGED) vmp_mbar_wait(&vmp_bar, 0);
        cclear = __all_sync(VMP_FULL, vmp_const_clear(env, a.env.ns, a.env.nc, a.env.nb, lane, 32));
        cdone = true;
        ok = ok && cclear;
      }}
      const unsigned bad = __ballot_sync(VMP_FULL, inr && !ok);
      if (tag == 0) {{                       // first write to the workspace: begin kernel done?
        asm volatile("griddepcontrol.wait;" ::: "memory");
        tag = (1ull + __ldcg(a.dq + VMP_DQ_CALLS) % 65535ull) << 48;
      }}
      if (bad && lane == 0) {{
        const unsigned it = Wu == 32 ? (unsigned)ci + 1 : (32u * (unsigned)ci + __ffs(bad) - 1) / Wu + 1;
        atomicMax(a.fail + ei, 0x7fffffff - (int)it);
      }}
      if (round0) {{                         // publish the edge's remaining chunks
        const int chunks = (int)vmp_rake_chunks((unsigned)n, Wu);
        // rake positions grow with the chunk index, so no later chunk can fail
        // at an earlier iteration than one found here: a failed edge is finished
        const int cnt = bad ? 0 : chunks - 1;
        // VMP_EXP=keep1 / keep2: the warp keeps the edge's last chunk(s) for itself
        // (no pop, no slot).  Measured slower - 35.1 -> 37.0 / 38.9 us: every chunk
        // in the shared queue balances better - so 0 is the default
        const int want = max(cnt - VMP_DQ_KEEP, 0);
        unsigned long long base = 0;
        if (lane == 0) {{
          a.n_of[ei] = n;
          base = atomicAdd(state, (1ull << 40) + (unsigned long long)want) & M40;
        }}
        base = __shfl_sync(VMP_FULL, base, 0);
        const long long fit = max(0ll, min((long long)want, cap - (long long)base));
        for (long long jx = lane; jx < fit; jx += 32) {{
          const unsigned long long c = (unsigned long long)(jx + 1);
          ulonglong2 w;
          w.x = tag | ((c & 0x1ffffull) << 31) | (unsigned long long)ei;
          w.y = tag | ((c >> 17) << 31) | (unsigned long long)(unsigned)n;
          __stcg((ulonglong2 *)(a.slots + 2 * ((long long)base + jx)), w);
        }}
        if (fit < cnt) {{
          loc_e = ei;
          loc_n = n;
          loc_c = (int)fit + 1;
          loc_end = chunks;
        }}
      }}
    }}
{_TRACE_BLOCK.replace("t < VMP_TRACE_ITEMS", "t >= 0 && t < VMP_TRACE_ITEMS") if TRACE_ITEMS else ""}
  }}
  if (trace && lane == 0) {{
    trace[2 + warp] = vmp_gtime();
    atomicAdd(trace + 7, (unsigned long long)taken);
  }}
  if (STAGED && !cdone) vmp_mbar_wait(&vmp_bar, 0);   // no item evaluated: still retire the copy
  if (trace && threadIdx.x == 0) trace[6] = vmp_gtime();
}}
"""
    for prune in (0, 1):
        for staged in (0, 1):
            for stop in (0, 1):
                g = "true" if staged else "false"
                src += (f'extern "C" __global__ void __launch_bounds__({BLOCK}) '
                        f'vmp_validate_p{prune}_s{stop}_g{staged}(VmpValidateArgs a) '
                        f'{{ vmp_validate_body<{prune}, {stop}, {g}, 1>(a); }}\n')
                if staged:
                    for sp in SPLITS:
                        src += (f'extern "C" __global__ void __launch_bounds__({BLOCK}) '
                                f'vmp_validate_p{prune}_s{stop}_g1_x{sp}(VmpValidateArgs a) '
                                f'{{ vmp_validate_body<{prune}, {stop}, true, {sp}>(a); }}\n')
                if staged:                          # 256-thread CTAs for large staged envs
                    src += (f'extern "C" __global__ void __launch_bounds__({2 * BLOCK}) '
                            f'vmp_validate_p{prune}_s{stop}_g1_b{2 * BLOCK}(VmpValidateArgs a) '
                            f'{{ vmp_validate_body<{prune}, {stop}, true, 1, false, {2 * BLOCK}>(a); }}\n')
                if staged and stop == 1:            # two-pass broadphase, small batches
                    for sp in (1, SPLIT):
                        src += (f'extern "C" __global__ void __launch_bounds__({BLOCK}) '
                                f'vmp_validate_p{prune}_s1_g1_x{sp}t(VmpValidateArgs a) '
                                f'{{ vmp_validate_body<{prune}, 1, true, {sp}, true>(a); }}\n')
            for stop in (1, 2):
                src += (f'extern "C" __global__ void __launch_bounds__({BLOCK}) '
                        f'vmp_motion_p{prune}_s{stop}_g{staged}(VmpMotionArgs a) '
                        f'{{ vmp_motion_body<{prune}, {stop}, {"true" if staged else "false"}>(a); }}\n')
            if staged:
                # the hot rake variant, register-capped for MOTION_MIN_CTAS CTAs per
                # SM; the host uses it only when it compiled without local memory
                src += (f'extern "C" __global__ void __launch_bounds__({BLOCK}, {MOTION_MIN_CTAS}) '
                        f'vmp_motion_p{prune}_s2_g1_o(VmpMotionArgs a) '
                        f'{{ vmp_motion_body<{prune}, 2, true>(a); }}\n')
                src += (f'extern "C" __global__ void __launch_bounds__({BLOCK}, {MOTION_MIN_CTAS}) '
                        f'vmp_motion_p{prune}_s2_g1_o_ns(VmpMotionArgs a) '
                        f'{{ vmp_motion_body<{prune}, 2, true, true>(a); }}\n')
    return src


def generate_source(program, pairs=None, name: str = "robot") -> str:
    """Complete NVRTC translation unit for one robot (self-contained)."""
    lay = derive_layout(program, pairs)
    abi = (CSRC / "vmp_abi.h").read_text()
    dev = (CSRC / "vmp_device.cuh").read_text()
    fk = _fk_lines(program)
    fk_macro = " \\\n  ".join(fk) if fk else ""
    const_defs = []
    values = np.asarray(program.values)
    for s in lay.const_spheres:          # constant centres, in the environment frame
        for axis, op, o in zip("XYZ", s.xyz, lay.home):
            const_defs.append(f"#define VMP_C{s.slot}{axis} {f32_literal(values[op] - o)}")
    # the environment frame the collision kernels assume (read by vmp_robot_load)
    const_defs.append('extern "C" __device__ const float vmp_home[3] = {'
                      + ", ".join(f32_literal(o) for o in lay.home) + "};")
    parts = [
        f"// generated by paper_2309_14545_b200.codegen v{CODEGEN_VERSION}",
        f"// dof={lay.dof} ops={lay.n_ops} markers={lay.n_markers} fine={len(lay.fine)} "
        f"const={len(lay.const_spheres)} pairs={len(lay.pairs)}",
        abi, dev,
        f"#define VMP_FK_BODY \\\n  {fk_macro}",
        "\n".join(const_defs),
    ]
    if lay.has_cc:
        parts.append(_const_check(lay))
        parts.append(_state_function(lay, program))
    parts.append(_kernels(lay, program))
    return "\n".join(parts) + "\n"


def source_key(source: str) -> str:
    return hashlib.sha256(source.encode()).hexdigest()[:24]


def algorithmic_flops(program, pairs, counts) -> dict:
    """Reference dense work per configuration.

    F = #MUL + #ADD + #SUB  +  N_fine * (8 ks + 20 kc + 26 kb)  +  8 * N_pairs
    (NEG and sin/cos not counted; coarse tests are pruning overhead).
    """
    kinds = np.asarray(program.kinds)
    f_fk = int(np.sum((kinds == MUL) | (kinds == ADD) | (kinds == SUB)))
    lay = derive_layout(program, pairs)
    ks, kc, kb = counts
    n_fine = len(lay.fine)
    f_env = n_fine * (8 * ks + 20 * kc + 26 * kb)
    f_self = 8 * len(lay.pairs)
    return {"fk": f_fk, "env": f_env, "self": f_self, "total": f_fk + f_env + f_self,
            "n_fine": n_fine, "n_pairs": len(lay.pairs),
            "n_const_fine": len(lay.const_spheres)}
