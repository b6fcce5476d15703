"""Host-side logic that needs no GPU: lanes helpers, documents, errors,
workload calibration, and the multi-rank sharding (gloo, world_size 2)."""

import os
import socket

import numpy as np
import pytest

from paper_2309_14545_b200 import (ConfigBlock, EnvironmentFormatError, aos_from_soa, as_config,
                                   interpolate_lanes, l2_distance, load_environment, load_robot,
                                   soa_from_aos, workloads)
from paper_2309_14545_b200.collision import CapsuleObstacle, environment_to_doc, parse_environment
from paper_2309_14545_b200.sharding import shard_range


def cfg(*v):
    return np.asarray(v, dtype=np.float32)


class TestLanes:
    def test_padding_replicates_lane_zero(self):
        block = soa_from_aos([cfg(1, 2), cfg(3, 4)], width=4)
        assert block.data.tolist() == [[1, 3, 1, 1], [2, 4, 2, 2]]
        assert [q.tolist() for q in aos_from_soa(block)] == [[1, 2], [3, 4]]

    def test_errors(self):
        with pytest.raises(ValueError):
            soa_from_aos([])
        with pytest.raises(ValueError):
            soa_from_aos([cfg(1, 2), cfg(1, 2, 3)])
        with pytest.raises(ValueError):
            soa_from_aos([cfg(0.0)] * 3, width=2)
        with pytest.raises(ValueError):
            ConfigBlock(2, 4, np.zeros((2, 3), np.float32), 1)
        with pytest.raises(ValueError):
            as_config([0.0, np.inf])

    def test_interpolation_and_distance(self):
        assert interpolate_lanes(cfg(0, 0), cfg(2, 4), np.asarray([0.5])).data[:, 0].tolist() == [1, 2]
        assert l2_distance(cfg(0, 0), cfg(3, 4)) == pytest.approx(5.0)
        with pytest.raises(ValueError):
            l2_distance(cfg(0, 0), cfg(1, 2, 3))


class TestDocuments:
    def test_cylinder_becomes_capsule(self):
        env = load_environment("primitives:\n  - {kind: cylinder, p0: [0,0,0], p1: [0,0,1], radius: 0.2}\n")
        assert isinstance(env.primitives[0], CapsuleObstacle)

    def test_rejections(self):
        with pytest.raises(EnvironmentFormatError, match="unknown primitive"):
            load_environment("primitives:\n  - {kind: torus, radius: 1.0}\n")
        with pytest.raises(EnvironmentFormatError, match="orthonormal"):
            load_environment("primitives:\n  - {kind: cuboid, center: [0,0,0], half_extents: [1,1,1],"
                             " rotation: [[2,0,0],[0,1,0],[0,0,1]]}\n")
        with pytest.raises(EnvironmentFormatError):
            load_environment("primitives:\n  - {kind: sphere, center: [0, 0, 0], radius: 0}\n")
        with pytest.raises(EnvironmentFormatError):
            load_environment("primitives:\n  - {kind: sphere, center: [0, 0], radius: 1}\n")
        assert load_environment("name: void\n").primitives == []

    def test_doc_round_trip(self):
        env = workloads.config4(8).env
        back = parse_environment(environment_to_doc(env))
        assert environment_to_doc(back) == environment_to_doc(env)

    def test_rpy_rotation(self):
        env = load_environment("primitives:\n  - {kind: cuboid, center: [0,0,0], half_extents: [1,1,1],"
                               " rpy: [0.3, -0.2, 1.1]}\n")
        r = env.primitives[0].rotation
        cr, sr, cp, sp, cy, sy = (np.cos(0.3), np.sin(0.3), np.cos(-0.2), np.sin(-0.2),
                                  np.cos(1.1), np.sin(1.1))
        expect = np.array([[cy * cp, cy * sp * sr - sy * cr, cy * sp * cr + sy * sr],
                           [sy * cp, sy * sp * sr + cy * cr, sy * sp * cr - cy * sr],
                           [-sp, cp * sr, cp * cr]])
        assert np.allclose(r, expect, atol=1e-15)


class TestWorkloads:
    def test_standins(self):
        dims = {n: load_robot(n).dof for n in ("arm7", "fetch_standin", "baxter_standin")}
        assert dims == {"arm7": 7, "fetch_standin": 8, "baxter_standin": 14}
        assert load_robot("panda") is load_robot("arm7")

    def test_keepout_rule(self):
        env = workloads.config3(8).env
        for p in env.primitives:
            if hasattr(p, "half_extents"):
                c, bound = p.center, float(np.linalg.norm(p.half_extents))
            elif hasattr(p, "p0"):
                c = 0.5 * (p.p0 + p.p1)
                bound = 0.5 * float(np.linalg.norm(p.p1 - p.p0)) + p.radius
            else:
                c, bound = p.center, p.radius
            assert np.hypot(c[0], c[1]) - bound >= workloads.KEEPOUT["fetch_standin"] - 1e-12

    def test_deterministic_and_shaped(self):
        a, b = workloads.config1(1024), workloads.config1(1024)
        assert np.array_equal(a.q, b.q) and a.q.shape == (7, 1024) and a.q.dtype == np.float32
        lims = load_robot("arm7").limits
        assert (a.q >= lims[:, :1].astype(np.float32)).all() and (a.q <= lims[:, 1:].astype(np.float32)).all()
        mw = workloads.config2()
        assert mw.starts.shape == (4096, 7) and mw.resolution == 1 / 32
        assert env_counts(workloads.config4(8).env) == (0, 16, 49)


def env_counts(env):
    return env.counts()


class TestSharding:
    @pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (31, 2), (100, 3), (4096, 8), (1 << 20, 7)])
    def test_ranges_partition(self, n, world):
        seen = []
        for r in range(world):
            lo, hi = shard_range(n, r, world)
            assert lo % 32 == 0 or lo == n
            seen.extend(range(lo, hi))
        assert seen == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    from paper_2309_14545_b200.sharding import validate_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    items = np.arange(n)

    def local(chunk):           # stand-in for the device kernel: valid iff item % 3 != 0
        bits = np.zeros(((len(chunk) + 31) // 32) * 32, dtype=np.uint8)
        bits[: len(chunk)] = (chunk % 3 != 0)
        words = np.packbits(bits, bitorder="little").view(np.uint32).astype(np.int64)
        return torch.tensor(words.astype(np.uint32).view(np.int32))

    out, _ = validate_sharded(local, items, rank, world)
    q.put((rank, out.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [1000, 4096])
def test_gloo_two_rank_gather(n):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = np.arange(n) % 3 != 0
    for r in range(2):
        bits = np.unpackbits(results[r].view(np.uint8), bitorder="little")[:n].astype(bool)
        assert np.array_equal(bits, expect)


def test_leading_dimension_ignores_size_one_strides():
    """A (1, N) batch made from an (N, 1) array keeps numpy's arbitrary
    stride for the size-1 dimension; the C ABI must get ld = N (this broke
    1-dof robots: reference test_planners.py::TestPrm sealed pendulum)."""
    import torch
    from paper_2309_14545_b200.runtime import ld
    one_row = torch.from_numpy(np.ascontiguousarray(np.zeros((64, 1), np.float32).T))
    assert one_row.shape == (1, 64) and ld(one_row) == 64
    assert ld(torch.zeros((3, 10))[:, :7]) == 10
    assert ld(torch.zeros((1, 5))) == 5


def test_rake_parameter_float32_division_equals_float64_quotient():
    """vmp_rake_param uses the IEEE float32 quotient for n < 2^24 in place of
    float32(i / n) taken in float64 (reference motion.py:69-70); double
    rounding cannot differ there (csrc/vmp_device.cuh).  Exhaustive for
    n <= 1500, 10^6 random pairs up to 2^24."""
    for n in range(1, 1501):
        i = np.arange(1, n + 1)
        assert np.array_equal((i / n).astype(np.float32),
                              i.astype(np.float32) / np.float32(n))
    rng = np.random.default_rng(7)
    n = rng.integers(1, 1 << 24, size=1_000_000)
    i = (rng.random(n.size) * n).astype(np.int64) + 1
    assert np.array_equal((i / n).astype(np.float32), i.astype(np.float32) / n.astype(np.float32))
