"""Kinematics tracing compiler: sphere-centre forward kinematics as a scalar op DAG.

Host-side, run once per robot (SURVEY.md §2 "Tracing compiler", scope ★(in)).
The op DAG is the intermediate representation that ``codegen.py`` lowers to a
straight-line sm_100a kernel, so it must be *the same* DAG the reference
builds: node creation order decides CSE outcomes and the scheduled op order.
tests/test_compiler_golden.py pins the optimized graphs against listings
generated from the reference (tests/golden/programs.json).

Reference interface followed (pkg/src/vecmp/trace.py):
  * op kinds / SphereKey / TraceGraph           trace.py:28-97
  * ``evaluate_graph`` (float64 semantics)      trace.py:100-137
  * ``rpy_to_matrix``  Rz(yaw) Ry(pitch) Rx(roll) trace.py:140-150
  * ``trace_kinematics`` (naive emission: every product and sum, including
    products with constant 0/1; Rodrigues for non-axis-aligned joints)
                                                 trace.py:153-264
  * ``optimize_graph`` (const fold, identities, double negation, CSE with
    canonical commutative operands, dead-node elimination) trace.py:273-379
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from .robot import KinematicTree, SphereModel

CONST, INPUT, ADD, SUB, MUL, NEG, SIN, COS = range(8)
KIND_NAMES = ("const", "input", "add", "sub", "mul", "neg", "sin", "cos")
UNARY_KINDS = (NEG, SIN, COS)

COARSE = "coarse"
FINE = "fine"


class SphereKey(NamedTuple):
    link: int
    level: str
    index: int


@dataclass
class TraceGraph:
    """Append-only scalar op arena; ``a``/``b`` are operand node ids (-1 = none)."""

    dof: int
    kinds: list = field(default_factory=list)
    a: list = field(default_factory=list)
    b: list = field(default_factory=list)
    values: list = field(default_factory=list)
    outputs: dict = field(default_factory=dict)
    radii: dict = field(default_factory=dict)

    def __len__(self) -> int:
        return len(self.kinds)

    def _node(self, kind: int, a: int = -1, b: int = -1, value: float = 0.0) -> int:
        size = len(self.kinds)
        if a >= size or b >= size:
            raise ValueError("operand must reference an earlier node")
        self.kinds.append(kind)
        self.a.append(a)
        self.b.append(b)
        self.values.append(value)
        return size

    def const(self, value: float) -> int:
        return self._node(CONST, value=float(value))

    def input(self, joint: int) -> int:
        if joint < 0 or joint >= self.dof:
            raise ValueError(f"joint index {joint} out of range for dof {self.dof}")
        return self._node(INPUT, value=float(joint))

    def add(self, x: int, y: int) -> int:
        return self._node(ADD, x, y)

    def sub(self, x: int, y: int) -> int:
        return self._node(SUB, x, y)

    def mul(self, x: int, y: int) -> int:
        return self._node(MUL, x, y)

    def neg(self, x: int) -> int:
        return self._node(NEG, x)

    def sin(self, x: int) -> int:
        return self._node(SIN, x)

    def cos(self, x: int) -> int:
        return self._node(COS, x)


_F64_UNARY = {NEG: np.negative, SIN: np.sin, COS: np.cos}
_F64_BINARY = {ADD: np.add, SUB: np.subtract, MUL: np.multiply}


def evaluate_graph(g: TraceGraph, q: np.ndarray) -> dict:
    """Double-precision evaluation of every output (reference trace.py:100-137).

    ``q`` is (dof,) or (n, dof); outputs are (3,) or (n, 3) positions.
    """
    batch = np.asarray(q, dtype=np.float64)
    scalar = batch.ndim == 1
    if scalar:
        batch = batch[None, :]
    if batch.shape[1] != g.dof:
        raise ValueError(f"configuration dim {batch.shape[1]} != dof {g.dof}")
    vals = np.empty((len(g), batch.shape[0]), dtype=np.float64)
    for i, kind in enumerate(g.kinds):
        if kind == CONST:
            vals[i] = g.values[i]
        elif kind == INPUT:
            vals[i] = batch[:, int(g.values[i])]
        elif kind in _F64_BINARY:
            _F64_BINARY[kind](vals[g.a[i]], vals[g.b[i]], out=vals[i])
        else:
            _F64_UNARY[kind](vals[g.a[i]], out=vals[i])
    result = {}
    for key, ids in g.outputs.items():
        pos = np.stack([vals[k] for k in ids], axis=-1)
        result[key] = pos[0] if scalar else pos
    return result


def rpy_to_matrix(rpy) -> np.ndarray:
    """Fixed-axis roll/pitch/yaw: Rz(yaw) @ Ry(pitch) @ Rx(roll)."""
    roll, pitch, yaw = (float(v) for v in rpy)
    sr, cr = math.sin(roll), math.cos(roll)
    sp, cp = math.sin(pitch), math.cos(pitch)
    sy, cy = math.sin(yaw), math.cos(yaw)
    return np.array([
        [cy * cp, cy * sp * sr - sy * cr, cy * sp * cr + sy * sr],
        [sy * cp, sy * sp * sr + cy * cr, sy * sp * cr - cy * sr],
        [-sp, cp * sr, cp * cr],
    ])


class _Emitter:
    """Symbolic 3x3 / 3-vector algebra over graph node ids.

    The emission order of every helper is part of the contract: it matches
    the reference's naive builder node for node (trace.py:153-189), which is
    what makes the optimized graphs identical.
    """

    def __init__(self, g: TraceGraph):
        self.g = g

    def const_mat(self, m) -> list:
        return [[self.g.const(m[r][c]) for c in range(3)] for r in range(3)]

    def const_vec(self, v) -> list:
        return [self.g.const(v[r]) for r in range(3)]

    def dot3(self, row, col) -> int:
        g = self.g
        first = g.mul(row[0], col[0])
        second = g.mul(row[1], col[1])
        acc = g.add(first, second)
        return g.add(acc, g.mul(row[2], col[2]))

    def matmul(self, lhs, rhs) -> list:
        g = self.g
        out = []
        for r in range(3):
            row = []
            for c in range(3):
                terms = [g.mul(lhs[r][k], rhs[k][c]) for k in range(3)]
                row.append(g.add(g.add(terms[0], terms[1]), terms[2]))
            out.append(row)
        return out

    def matvec(self, m, v) -> list:
        return [self.dot3(m[r], v) for r in range(3)]

    def vadd(self, u, v) -> list:
        return [self.g.add(u[r], v[r]) for r in range(3)]

    def joint_rotation(self, axis: np.ndarray, s: int, c: int) -> list:
        g = self.g
        aligned = _axis_alignment(axis)
        if aligned is not None:
            k, positive = aligned
            sn = s if positive else g.neg(s)
            one, zero = g.const(1.0), g.const(0.0)
            if k == 0:
                return [[one, zero, zero], [zero, c, g.neg(sn)], [zero, sn, c]]
            if k == 1:
                return [[c, zero, sn], [zero, one, zero], [g.neg(sn), zero, c]]
            return [[c, g.neg(sn), zero], [sn, c, zero], [zero, zero, one]]
        ax, ay, az = (float(v) for v in axis)
        skew = np.array([[0.0, -az, ay], [az, 0.0, -ax], [-ay, ax, 0.0]])
        outer = np.outer(axis, axis)
        ident = np.eye(3)
        versine = g.sub(g.const(1.0), c)
        rows = []
        for r in range(3):
            row = []
            for col in range(3):
                term = g.mul(c, g.const(ident[r][col]))
                term = g.add(term, g.mul(s, g.const(skew[r][col])))
                term = g.add(term, g.mul(versine, g.const(outer[r][col])))
                row.append(term)
            rows.append(row)
        return rows


def _axis_alignment(axis: np.ndarray):
    """(component, positive) when ``axis`` is +-x/y/z within 1e-9, else None."""
    for k in range(3):
        for sign in (1.0, -1.0):
            unit = np.zeros(3)
            unit[k] = sign
            if np.linalg.norm(axis - unit) < 1e-9:
                return k, sign > 0
    return None


def trace_kinematics(tree: KinematicTree, model: SphereModel) -> TraceGraph:
    """Trace world positions of every coarse and fine sphere (reference trace.py:228-264)."""
    g = TraceGraph(dof=tree.dof)
    em = _Emitter(g)
    frames = {tree.root: (em.const_mat(np.eye(3)), em.const_vec(np.zeros(3)))}
    for joint in tree.joints:
        if joint.parent not in frames:
            raise ValueError(f"joint {joint.name!r} parent not reachable from root")
        rot_p, pos_p = frames[joint.parent]
        rot = em.matmul(rot_p, em.const_mat(rpy_to_matrix(joint.rpy)))
        pos = em.vadd(em.matvec(rot_p, em.const_vec(joint.xyz)), pos_p)
        if joint.kind == "fixed":
            frames[joint.child] = (rot, pos)
            continue
        q = g.input(joint.input_index)
        if joint.kind == "prismatic":
            shift = []
            for component in joint.axis:
                shift.append(g.mul(g.const(float(component)), q))
            frames[joint.child] = (rot, em.vadd(em.matvec(rot, shift), pos))
        else:
            s, c = g.sin(q), g.cos(q)
            frames[joint.child] = (em.matmul(rot, em.joint_rotation(joint.axis, s, c)), pos)

    for link, spheres in enumerate(model.fine):
        if not spheres:
            continue
        if link not in frames:
            raise ValueError(f"link {tree.links[link]!r} not reachable from root")
        rot, pos = frames[link]
        for level, group in ((COARSE, [model.coarse[link]]), (FINE, spheres)):
            for idx, sphere in enumerate(group):
                centre = em.vadd(em.matvec(rot, em.const_vec(sphere.center)), pos)
                key = SphereKey(link=link, level=level, index=idx)
                g.outputs[key] = (centre[0], centre[1], centre[2])
                g.radii[key] = float(sphere.radius)
    return g


class _Interner:
    """Hash-consing node factory for the optimizer (CSE)."""

    def __init__(self, dof: int):
        self.graph = TraceGraph(dof=dof)
        self.table: dict = {}

    def make(self, kind: int, a: int = -1, b: int = -1, value: float = 0.0) -> int:
        if kind in (ADD, MUL) and a > b:
            a, b = b, a
        key = (kind, a, b, np.float64(value).tobytes())
        hit = self.table.get(key)
        if hit is None:
            hit = self.table[key] = self.graph._node(kind, a, b, value)
        return hit

    def is_const(self, n: int) -> bool:
        return n >= 0 and self.graph.kinds[n] == CONST

    def value(self, n: int) -> float:
        return self.graph.values[n]


def _rewrite(ir: _Interner, kind: int, a: int, b: int) -> int:
    """Apply the reference's rewrite rules in order; fall back to a fresh node."""
    ka, kb = ir.is_const(a), ir.is_const(b)
    va = ir.value(a) if ka else None
    vb = ir.value(b) if kb else None
    if kind == ADD:
        if ka and kb:
            return ir.make(CONST, value=va + vb)
        if ka and va == 0.0:
            return b
        if kb and vb == 0.0:
            return a
    elif kind == SUB:
        if ka and kb:
            return ir.make(CONST, value=va - vb)
        if kb and vb == 0.0:
            return a
        if ka and va == 0.0:
            return ir.make(NEG, b)
        if a == b:
            return ir.make(CONST, value=0.0)
    elif kind == MUL:
        if ka and kb:
            return ir.make(CONST, value=va * vb)
        if (ka and va == 0.0) or (kb and vb == 0.0):
            return ir.make(CONST, value=0.0)
        if ka and va == 1.0:
            return b
        if kb and vb == 1.0:
            return a
    elif kind == NEG:
        if ka:
            return ir.make(CONST, value=-va)
        if ir.graph.kinds[a] == NEG:
            return ir.graph.a[a]
    elif kind == SIN:
        if ka:
            return ir.make(CONST, value=math.sin(va))
    elif kind == COS:
        if ka:
            return ir.make(CONST, value=math.cos(va))
    return ir.make(kind, a, b)


def optimize_graph(g: TraceGraph) -> TraceGraph:
    """Semantics-preserving simplification (reference trace.py:273-379).

    Every rewrite is value-identical in float64; the pass never grows the
    graph and is idempotent.
    """
    ir = _Interner(g.dof)
    mapping: list[int] = []
    for i, kind in enumerate(g.kinds):
        if kind in (CONST, INPUT):
            mapping.append(ir.make(kind, value=g.values[i]))
            continue
        a = mapping[g.a[i]]
        b = mapping[g.b[i]] if g.b[i] >= 0 else -1
        mapping.append(_rewrite(ir, kind, a, b))

    mid = ir.graph
    reachable = np.zeros(len(mid), dtype=bool)
    frontier = [mapping[n] for ids in g.outputs.values() for n in ids]
    while frontier:
        n = frontier.pop()
        if reachable[n]:
            continue
        reachable[n] = True
        frontier.extend(x for x in (mid.a[n], mid.b[n]) if x >= 0 and not reachable[x])

    final = TraceGraph(dof=g.dof)
    renumber = np.full(len(mid), -1, dtype=np.int64)
    for n in np.flatnonzero(reachable):
        n = int(n)
        a = int(renumber[mid.a[n]]) if mid.a[n] >= 0 else -1
        b = int(renumber[mid.b[n]]) if mid.b[n] >= 0 else -1
        renumber[n] = final._node(mid.kinds[n], a, b, mid.values[n])
    for key, ids in g.outputs.items():
        final.outputs[key] = tuple(int(renumber[mapping[n]]) for n in ids)
    final.radii = dict(g.radii)
    return final
