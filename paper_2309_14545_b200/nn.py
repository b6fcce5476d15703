"""Exact nearest-neighbour index on the device.

Mirrors the reference ``NNIndex`` (pkg/src/vecmp/nn.py:18-69): same
constructor, ``insert`` / ``__len__`` / ``nearest`` / ``k_nearest``, same
errors, same answers - float32 distances summed in joint order and rooted
(nn.py:45-51), ascending with ties to the first-inserted point (the stable
argsort, nn.py:67-69).  Points live in HBM as a (dim, capacity) float32 SoA
buffer; inserts are staged on the host and flushed in one copy before the
next query.  ``k_nearest_many`` answers a batch of queries in one launch,
each optionally restricted to a prefix of the index (a query issued
"between" inserts, as the PRM round does).

k <= 32 (dim <= 64) runs the query-tiled top-k kernel (vmp_knn); larger k or
dim sorts the full distance row (vmp_nn_distances, any dim up to 12,288)
with a stable device sort - same answers, no dimension limit in practice
(the reference's NNIndex has none).
"""

from __future__ import annotations

import numpy as np

from . import runtime
from ._native import VMP_KNN_MAX_DIM, VMP_KNN_MAX_K

NN_MAX_DIM = 12288          # vmp_nn_distances stages a query row in shared memory


class NNIndex:
    def __init__(self, dim: int):
        if dim < 1:
            raise ValueError("dim must be >= 1")
        if dim > NN_MAX_DIM:
            raise ValueError(f"dim must be <= {NN_MAX_DIM}")
        self.dim = dim
        self._payloads: list = []
        self._ids: set = set()
        self._pending: list[np.ndarray] = []
        self._points = None                  # (dim, capacity) device tensor
        self._flushed = 0

    def __len__(self) -> int:
        return len(self._payloads)

    def _vec(self, q) -> np.ndarray:
        qv = np.asarray(q, dtype=np.float32).reshape(-1)
        if qv.shape[0] != self.dim:
            raise ValueError(f"dimension mismatch: {qv.shape[0]} vs {self.dim}")
        return qv

    def insert(self, q, payload) -> None:
        qv = self._vec(q)
        if payload in self._ids:
            raise ValueError(f"duplicate payload id: {payload!r}")
        self._pending.append(qv.copy())
        self._payloads.append(payload)
        self._ids.add(payload)

    def insert_many(self, qs, payloads) -> None:
        """Insert rows of ``qs`` in order (same checks as ``insert``)."""
        for q, p in zip(np.asarray(qs, dtype=np.float32).reshape(-1, self.dim), payloads):
            self.insert(q, p)

    def _flush(self):
        torch = runtime.require_cuda()
        n = len(self._payloads)
        cap = 0 if self._points is None else self._points.shape[1]
        if n > cap:
            grown = torch.empty((self.dim, max(64, 2 * cap, n)), dtype=torch.float32,
                                device=torch.cuda.current_device())
            if self._flushed:
                grown[:, :self._flushed] = self._points[:, :self._flushed]
            self._points = grown
        if self._pending:
            block = torch.from_numpy(np.ascontiguousarray(np.stack(self._pending, axis=1)))
            self._points[:, self._flushed:n] = block.to(self._points.device)
            self._pending.clear()
            self._flushed = n
        return self._points

    def _device_query(self, qs, k: int, visible=None):
        torch = runtime.require_cuda()
        points = self._flush()
        n = len(self._payloads)
        qd = runtime.to_device(np.ascontiguousarray(qs, dtype=np.float32).reshape(-1, self.dim))
        vis = None if visible is None else torch.as_tensor(
            np.asarray(visible, dtype=np.int64)).to(qd.device)
        if k <= VMP_KNN_MAX_K and self.dim <= VMP_KNN_MAX_DIM:
            return runtime.knn_device(points, n, qd, k, vis)
        dist = runtime.nn_distances_device(points, n, qd)
        if vis is not None:
            cols = torch.arange(n, device=qd.device)
            dist = torch.where(cols[None, :] < vis[:, None], dist,
                               torch.full_like(dist, float("inf")))
        sd, si = torch.sort(dist, dim=1, stable=True)
        k = min(k, n)
        idx, sd = si[:, :k].to(torch.int32), sd[:, :k]
        if vis is not None:
            idx = torch.where(cols[:k][None, :] < vis[:, None], idx, torch.full_like(idx, -1))
        return idx, sd

    def nearest(self, q) -> tuple[object, float]:
        """Exact closest point's (payload, distance); first-inserted wins ties."""
        qv = self._vec(q)
        if not self._payloads:
            raise ValueError("nearest query on an empty index")
        idx, dist = self._device_query(qv[None, :], 1)
        i = int(idx[0, 0])
        return self._payloads[i], float(dist[0, 0])

    def k_nearest(self, q, k: int) -> list[tuple[object, float]]:
        """The k exact closest points, ascending distance (fewer if smaller)."""
        if k < 1:
            raise ValueError("k must be >= 1")
        qv = self._vec(q)
        if not self._payloads:
            raise ValueError("k_nearest query on an empty index")
        k = min(k, len(self._payloads))
        idx, dist = self._device_query(qv[None, :], k)
        idx, dist = idx[0].cpu().numpy(), dist[0].cpu().numpy()
        return [(self._payloads[int(i)], float(d)) for i, d in zip(idx, dist) if i >= 0]

    def k_nearest_many(self, qs, k: int, visible=None):
        """Batched exact k-NN: (Q, k) int32 insertion indices (-1 = none) and
        float32 distances as numpy arrays; query q only sees the first
        ``visible[q]`` points when given."""
        if k < 1:
            raise ValueError("k must be >= 1")
        qs = np.asarray(qs, dtype=np.float32).reshape(-1, self.dim)
        if len(qs) == 0 or not self._payloads:
            return (np.full((len(qs), k), -1, np.int32),
                    np.full((len(qs), k), np.inf, np.float32))
        idx, dist = self._device_query(qs, k, visible)
        idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
        if idx.shape[1] < k:
            pad = k - idx.shape[1]
            idx = np.pad(idx, ((0, 0), (0, pad)), constant_values=-1)
            dist = np.pad(dist, ((0, 0), (0, pad)), constant_values=np.inf)
        return idx, dist
