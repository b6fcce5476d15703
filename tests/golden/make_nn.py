"""Golden fixtures for the exact k-NN scan, from the REFERENCE NNIndex
(nn.py:18-69; build container only).

    python tests/golden/make_nn.py     -> tests/golden/nn.npz

Seeded point sets (some on a coarse grid, so distance ties occur) and
queries; records the reference k_nearest payload order and distances.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from vecmp.nn import NNIndex  # noqa: E402

CASES = ((1, 1, 0), (2, 6, 0), (3, 100, 0), (7, 1000, 0), (14, 257, 0), (2, 300, 1), (7, 500, 1),
         (1, 64, 1))
KS = (1, 5, 32, 50)


def main() -> None:
    out = {}
    rng = np.random.default_rng(2309)
    for c, (dim, n, grid) in enumerate(CASES):
        pts = rng.normal(size=(n, dim))
        qs = rng.normal(size=(16, dim))
        if grid:                                     # coarse lattice -> many exact ties
            pts, qs = np.round(pts * 2) / 2, np.round(qs * 2) / 2
        pts, qs = pts.astype(np.float32), qs.astype(np.float32)
        idx = NNIndex(dim)
        for i, p in enumerate(pts):
            idx.insert(p, i)
        out[f"points_{c}"], out[f"queries_{c}"] = pts, qs
        for k in KS:
            res = [idx.k_nearest(q, k) for q in qs]
            out[f"index_{c}_k{k}"] = np.asarray([[p for p, _ in r] for r in res], np.int64)
            out[f"dist_{c}_k{k}"] = np.asarray([[d for _, d in r] for r in res], np.float32)
        out[f"nearest_{c}"] = np.asarray([idx.nearest(q)[0] for q in qs], np.int64)
    np.savez_compressed(HERE / "nn.npz", **out)
    print("wrote", HERE / "nn.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
