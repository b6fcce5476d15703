"""Exact k-NN scan against the reference NNIndex.

tests/golden/nn.npz holds the reference's own k_nearest / nearest answers
(nn.py:45-69) on seeded point sets, half of them on a coarse lattice so
distance ties are common (make_nn.py).  The oracle restatement is pinned to
those on CPU; the device index must return the identical order (ties to the
first-inserted point) and bit-identical float32 distances.
"""

import numpy as np
import pytest

import golden_io
import vecmp_oracle as O

FX = golden_io.load("nn")
CASES = sorted({int(k.split("_")[1]) for k in FX.files if k.startswith("points_")})
KS = (1, 5, 32, 50)


@pytest.mark.parametrize("c", CASES)
def test_oracle_matches_reference_golden(c):
    pts, qs = FX[f"points_{c}"], FX[f"queries_{c}"]
    soa = np.ascontiguousarray(pts.T)
    for k in KS:
        for qi, q in enumerate(qs):
            idx, dist = O.nn_k_nearest(soa, q, k)
            assert idx.tolist() == FX[f"index_{c}_k{k}"][qi].tolist()
            assert np.array_equal(dist, FX[f"dist_{c}_k{k}"][qi])


def _index(pts):
    from paper_2309_14545_b200.nn import NNIndex
    idx = NNIndex(pts.shape[1])
    for i, p in enumerate(pts):
        idx.insert(p, i)
    return idx


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES)
def test_device_index_matches_reference(cuda, c):
    pts, qs = FX[f"points_{c}"], FX[f"queries_{c}"]
    idx = _index(pts)
    for k in KS:
        for qi, q in enumerate(qs):
            got = idx.k_nearest(q, k)
            assert [p for p, _ in got] == FX[f"index_{c}_k{k}"][qi].tolist(), (c, k, qi)
            assert np.array_equal(np.asarray([d for _, d in got], np.float32),
                                  FX[f"dist_{c}_k{k}"][qi])
        many, dist = idx.k_nearest_many(qs, k)
        expect = FX[f"index_{c}_k{k}"]
        assert np.array_equal(many[:, :expect.shape[1]], expect)
        assert (many[:, expect.shape[1]:] == -1).all()
    assert [idx.nearest(q)[0] for q in qs] == FX[f"nearest_{c}"].tolist()


@pytest.mark.gpu
def test_device_index_errors_mirror_reference(cuda):
    from paper_2309_14545_b200.nn import NNIndex
    with pytest.raises(ValueError):
        NNIndex(0)
    idx = NNIndex(2)
    with pytest.raises(ValueError):
        idx.nearest(np.zeros(2, np.float32))
    with pytest.raises(ValueError):
        idx.k_nearest(np.zeros(2, np.float32), 1)
    idx.insert(np.zeros(2, np.float32), "a")
    with pytest.raises(ValueError, match="duplicate"):
        idx.insert(np.ones(2, np.float32), "a")
    with pytest.raises(ValueError):
        idx.insert(np.zeros(3, np.float32), "b")
    with pytest.raises(ValueError):
        idx.k_nearest(np.zeros(2, np.float32), 0)
    assert idx.nearest(np.ones(2, np.float32)) == ("a", pytest.approx(np.sqrt(2.0)))


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n,k", [(7, 100_000, 8), (14, 30_000, 32), (3, 5000, 64),
                                     (100, 3000, 5), (300, 2000, 40)])
def test_batched_prefix_queries_match_oracle(cuda, dim, n, k):
    """k_nearest_many with per-query visible prefixes == the oracle on each prefix."""
    rng = np.random.default_rng(dim * 1000 + k)
    pts = (np.round(rng.uniform(-1, 1, size=(n, dim)) * 8) / 8).astype(np.float32)
    qs = (np.round(rng.uniform(-1, 1, size=(64, dim)) * 8) / 8).astype(np.float32)
    visible = rng.integers(0, n + 1, size=len(qs))
    visible[:3] = (0, 1, n)
    idx = _index(pts)
    got, dist = idx.k_nearest_many(qs, k, visible=visible)
    soa = np.ascontiguousarray(pts.T)
    for qi, q in enumerate(qs):
        m = int(visible[qi])
        ei, ed = O.nn_k_nearest(soa[:, :m], q, k)
        assert got[qi, :len(ei)].tolist() == ei.tolist(), (qi, m)
        assert np.array_equal(dist[qi, :len(ei)], ed)
        assert (got[qi, len(ei):] == -1).all()


@pytest.mark.gpu
@pytest.mark.parametrize("dim,k", [(7, 8), (14, 32), (2, 1)])
def test_query_tiled_kernel_matches_oracle(cuda, dim, k):
    """>= 2,368 queries take the CTA-tiled kernel (shared point chunks, 4
    queries per warp, squared-distance filter); lattice points force ties."""
    rng = np.random.default_rng(dim + 100 * k)
    n, nq = 20_000, 3_000
    pts = (np.round(rng.uniform(-1, 1, size=(n, dim)) * 4) / 4).astype(np.float32)
    qs = (np.round(rng.uniform(-1, 1, size=(nq, dim)) * 4) / 4).astype(np.float32)
    visible = rng.integers(0, n + 1, size=nq)
    visible[:4] = (0, 1, 255, n)
    idx = _index(pts)
    got, dist = idx.k_nearest_many(qs, k, visible=visible)
    soa = np.ascontiguousarray(pts.T)
    for qi in list(range(8)) + list(rng.choice(nq, 200, replace=False)):
        m = int(visible[qi])
        ei, ed = O.nn_k_nearest(soa[:, :m], qs[qi], k)
        assert got[qi, :len(ei)].tolist() == ei.tolist(), (qi, m)
        assert np.array_equal(dist[qi, :len(ei)], ed)
        assert (got[qi, len(ei):] == -1).all()
