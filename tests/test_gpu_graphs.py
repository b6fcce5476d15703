"""CUDA-graph fixed-size entry points give the same verdicts as the eager path."""

import numpy as np
import pytest

import vecmp_oracle as O
from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads
from paper_2309_14545_b200 import motion as M

pytestmark = pytest.mark.gpu


def test_motion_validator_graph_matches_eager_and_oracle(cuda):
    torch = cuda
    mw = workloads.config2()
    rob = load_robot(mw.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
    eager = runtime.unpack_bits(
        M.validate_motions(ctx, mw.starts, mw.goals, mw.resolution).cpu().numpy(), len(mw.starts))
    mv = M.MotionValidator(ctx, len(mw.starts), mw.resolution)
    hs = torch.from_numpy(mw.starts).pin_memory()
    hg = torch.from_numpy(mw.goals).pin_memory()
    for _ in range(5):                       # replays with fresh host inputs each time
        mv(hs, hg)
        assert mv.verdicts().tolist() == eager.tolist()
    # a different batch through the same graph
    rng = np.random.default_rng(9)
    idx = rng.permutation(len(mw.starts))
    mv(mw.starts[idx], mw.goals[idx])
    assert mv.verdicts().tolist() == eager[idx].tolist()
    ob = O.Obstacles(mw.env.primitives)
    for i in range(0, len(mw.starts), 97):
        _, v = O.edge_all_states(rob.program, rob.pairs, ob, mw.starts[i], mw.goals[i], mw.resolution)
        assert bool(v.all()) == bool(eager[i])


def test_motion_pipeline_overlapped_batches(cuda):
    torch = cuda
    mw = workloads.config2()
    rob = load_robot(mw.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
    E = 1024
    batches = []
    rng = np.random.default_rng(4)
    for _ in range(6):
        idx = rng.choice(len(mw.starts), E, replace=False)
        batches.append((torch.from_numpy(mw.starts[idx]).pin_memory(),
                        torch.from_numpy(mw.goals[idx]).pin_memory()))
    expect = [runtime.unpack_bits(M.validate_motions(ctx, s, g, mw.resolution).cpu().numpy(), E)
              for s, g in batches]
    for depth in (2, 3):
        pipe = M.MotionPipeline(ctx, E, mw.resolution, depth=depth)
        inflight = []
        for k, (s, g) in enumerate(batches + batches):        # slots are reused
            inflight.append((k, pipe.submit(s, g)))
            if len(inflight) == depth:
                j, t = inflight.pop(0)
                got = runtime.unpack_bits(pipe.result(t), E)
                assert got.tolist() == expect[j % len(batches)].tolist()
        for j, t in inflight:
            assert runtime.unpack_bits(pipe.result(t), E).tolist() == \
                expect[j % len(batches)].tolist()
    # the intended use: ONE pair of pinned buffers refilled in place every step
    # (whole-step graphs keyed by the source pointers), then pageable numpy
    # batches (no graph for the copies) through the same pipeline
    pipe = M.MotionPipeline(ctx, E, mw.resolution, depth=2)
    hs, hg = torch.empty_like(batches[0][0]).pin_memory(), torch.empty_like(batches[0][1]).pin_memory()
    for j, (s, g) in enumerate(batches):
        hs.copy_(s)
        hg.copy_(g)
        assert runtime.unpack_bits(pipe.result(pipe.submit(hs, hg)), E).tolist() == expect[j].tolist()
    assert all(len(c) == 1 for c in pipe._step_graphs)
    for j, (s, g) in enumerate(batches):
        t = pipe.submit(s.numpy().copy(), g.numpy().copy())
        assert runtime.unpack_bits(pipe.result(t), E).tolist() == expect[j].tolist()


@pytest.mark.parametrize("early", [True, False])
def test_config_validator_graph(cuda, early):
    wl = workloads.config3(1 << 16)
    rob = load_robot(wl.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
    n = wl.q.shape[1]
    cv = ctx.batch_validator(n, early_exit=early)
    cv(wl.q)
    got = runtime.unpack_bits(cv().cpu().numpy(), n)
    assert np.array_equal(got, ctx.validate_configs(wl.q))
    q2 = workloads.uniform_configs(rob.limits, n, 77)
    cv(q2)
    assert np.array_equal(runtime.unpack_bits(cv().cpu().numpy(), n), ctx.validate_configs(q2))


@pytest.mark.parametrize("cfg", ["cfg1", "cfg4"])
@pytest.mark.parametrize("early", [True, False])
def test_split_kernel_matches_single_thread_kernel(cuda, cfg, early):
    """The small-batch split kernel (4 warps per 32 configurations, obstacles and
    self pairs partitioned) gives bit-identical verdict words."""
    torch = cuda
    wl = workloads.config1() if cfg == "cfg1" else workloads.config4(200_003)
    rob = load_robot(wl.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
    q = torch.from_numpy(wl.q).cuda()
    n = q.shape[1]
    words = {}
    for split in (True, False):
        words[split] = runtime.validate_device(ctx.module, ctx.device_env, q, n, q.stride(0),
                                               early_exit=early, split=split).cpu().numpy()
    assert np.array_equal(words[True], words[False])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg3", "cfg4"])
def test_every_kernel_variant_gives_the_same_words(cuda, cfg):
    """Single-thread / split, one-pass / two-pass broadphase, early exit /
    dense: six kernels, bit-identical verdict words (the product path picks
    among them by batch size and scene; the oracle checks the product path)."""
    torch = cuda
    n = 70_001
    wl = {"cfg1": workloads.config1, "cfg3": workloads.config3, "cfg4": workloads.config4}[cfg](n)
    rob = load_robot(wl.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
    q = torch.from_numpy(wl.q).cuda()
    ref = ctx.validate_batch(q).cpu().numpy()
    for kw in (dict(split=False), dict(split=True), dict(split=False, two_pass=True),
               dict(split=True, two_pass=True), dict(split=False, early_exit=False),
               dict(split=True, early_exit=False)):
        got = runtime.validate_device(ctx.module, ctx.device_env, q, n, q.stride(0), **kw)
        assert np.array_equal(got.cpu().numpy(), ref), kw


@pytest.mark.parametrize("cfg,n", [("cfg1", 65536), ("cfg3", 20000), ("cfg1", 1000)])
def test_config_stream_pdl_chain(cuda, cfg, n):
    """One graph of PDL-chained launches over distinct resident batches gives
    every batch the verdicts of its own standalone launch."""
    wl = workloads.config1(n) if cfg == "cfg1" else workloads.config3(n)
    rob = load_robot(wl.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
    batches = [workloads.uniform_configs(rob.limits, n, 900 + i) for i in range(7)]
    cs = ctx.stream_validator(n, len(batches))
    for i, q in enumerate(batches):
        cs.load(i, q)
    for _ in range(3):
        out = cs()
        for q, words in zip(batches, out):
            assert np.array_equal(words.cpu().numpy(), ctx.validate_batch(q).cpu().numpy())
