"""Experiment: per-batch time of the FK+CC kernels when batches stream back to
back (R distinct input copies whose total exceeds the L2, one launch each,
between two events) vs one flushed launch between events.

    VMP_EXP_SPLIT=1|2|4 python scripts/exp_stream.py [cfg1 cfg3 cfg4]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
L2 = 126 << 20


def streamed(launch, copies, reps=3):
    best = 1e9
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(copies):
            launch(i)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / copies)
    return best


def single(launch, reps=20):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        launch(0)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.mean(ts))


for key in sys.argv[1:] or ["cfg1"]:
    wl = {"cfg1": workloads.config1, "cfg3": workloads.config3, "cfg4": workloads.config4}[key]()
    rob = load_robot(wl.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
    n = wl.q.shape[1]
    copies = max(4, -(-2 * L2 // wl.q.nbytes))
    qs = [torch.from_numpy(wl.q).cuda() for _ in range(copies)]
    outs = [torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda") for _ in range(copies)]
    for tag, kw in (("prod", {}), ("dense", dict(early_exit=False)), ("prod_np", dict(prune=False)),
                    ("prod_pdl", dict(pdl=True))):
        def launch(i, kw=kw):
            runtime.validate_device(ctx.module, ctx.device_env, qs[i], n, n, out=outs[i], **kw)
        launch(0)
        # graphs: one captured launch per copy, replayed back to back
        graphs = []
        for i in range(copies):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                launch(i)
            graphs.append(g)
        ref = outs[0].clone()
        s_us = streamed(lambda i: graphs[i].replay(), copies)
        # all copies in ONE graph (consecutive launches get programmatic edges with pdl)
        gall = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gall):
            for i in range(copies):
                launch(i)
        s_all = streamed(lambda i: gall.replay() if i == 0 else None, copies)
        one = single(lambda i: graphs[i].replay())
        assert torch.equal(outs[1], ref)
        print(f"{key} {tag:8s} copies={copies:4d}  streamed {s_us:7.2f} us/batch  "
              f"one-graph {s_all:7.2f} us/batch  single flushed {one:7.2f} us", flush=True)
