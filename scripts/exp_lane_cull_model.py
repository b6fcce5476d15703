"""Model (CPU, numpy): narrowphase work of the batch FK+CC kernel under (a) the warp-vote
broadphase (an obstacle near ANY lane's ANY group -> every lane tests every sphere) and
(b) per-lane, per-group near lists (each lane pops its own near obstacles group by group;
a warp iterates max-over-lanes times).  Counts sphere-obstacle tests per warp.
    python scripts/exp_lane_cull_model.py cfg3|cfg4|cfg1 [n_configs]
"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import vecmp_oracle as O
from paper_2309_14545_b200 import load_robot, workloads, codegen

what = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
wl = {"cfg1": workloads.config1, "cfg3": workloads.config3, "cfg4": workloads.config4}[what](n)
rob = load_robot(wl.robot)
lay = codegen.derive_layout(rob.program, rob.pairs)
rows = O.rows_f64(rob.program, wl.q.astype(np.float64))
cent = O.marker_centres(rob.program, rows)            # (markers, 3, N)
fine_idx = [i for i, m in enumerate(rob.program.checks) if m.level == codegen.FINE]
dyn = lay.dynamic
groups = [dyn[i:i + 3] for i in range(0, len(dyn), 3)]
# obstacle bounding spheres
bc, br, kinds = [], [], []
for p in wl.env.primitives:
    k = O._kind(p)
    if k == "sphere": c, r = np.asarray(p.center, float), p.radius
    elif k == "capsule":
        p0, p1 = np.asarray(p.p0, float), np.asarray(p.p1, float); c, r = (p0 + p1) / 2, np.linalg.norm(p1 - p0) / 2 + p.radius
    else: c, r = np.asarray(p.center, float), np.linalg.norm(p.half_extents)
    bc.append(c); br.append(r); kinds.append(k)
bc, br = np.asarray(bc), np.asarray(br)
near = []                                             # per group: (K, N) bool
for g in groups:
    mid = g[len(g) // 2]
    cm = cent[fine_idx[mid.slot]]                     # (3, N)
    R = np.full(cm.shape[1], mid.radius)
    for s in g:
        if s is mid: continue
        R = np.maximum(R, np.linalg.norm(cent[fine_idx[s.slot]] - cm, axis=0) + s.radius)
    d = np.linalg.norm(cm[None] - bc[:, :, None], axis=1)     # (K, N)
    near.append(d <= R[None] + br[:, None])
near = np.asarray(near)                               # (G, K, N)
G, K, N = near.shape
W = N // 32
nw = near.reshape(G, K, W, 32)
sizes = np.asarray([len(g) for g in groups])
# (a) warp vote on min over groups
any_lane = nw.any(axis=(0, 3))                        # (K, W)
tests_a = any_lane.sum(axis=0) * len(dyn)             # sphere tests per warp (per lane)
# (b) per-lane per-group lists, per kind chunk of 32
order = sorted(range(K), key=lambda k: ["sphere", "capsule", "box"].index(kinds[k]))
tests_b = np.zeros(W); iters_b = np.zeros(W)
for kind in ("sphere", "capsule", "box"):
    ks = [k for k in order if kinds[k] == kind]
    for c0 in range(0, len(ks), 32):
        sel = ks[c0:c0 + 32]
        cnt = nw[:, sel].sum(axis=1)                  # (G, W, 32)
        mx = cnt.max(axis=2)                          # (G, W)
        iters_b += mx.sum(axis=0)
        tests_b += (mx * sizes[:, None]).sum(axis=0)
# (c) per-lane single mask (any group), all spheres
tests_c = np.zeros(W)
for kind in ("sphere", "capsule", "box"):
    ks = [k for k in order if kinds[k] == kind]
    for c0 in range(0, len(ks), 32):
        sel = ks[c0:c0 + 32]
        cnt = nw[:, sel].any(axis=0).sum(axis=0)      # (W, 32)
        tests_c += cnt.max(axis=1) * len(dyn)
print(f"{what}: {len(dyn)} dynamic spheres, {G} groups, {K} obstacles, {W} warps")
print(f"  per-lane P(group near obstacle) = {near.mean():.4f}; per-lane near pairs = {near.sum(axis=(0, 1)).mean():.2f}")
print(f"  (a) warp vote: {any_lane.mean() * 100:.1f}% of (obstacle, warp) near; sphere tests per lane-slot per warp = {tests_a.mean():.1f}")
print(f"  (b) per-lane per-group lists: iterations per warp = {iters_b.mean():.1f}, sphere tests = {tests_b.mean():.1f}")
print(f"  (c) per-lane any-group lists: sphere tests = {tests_c.mean():.1f}")
