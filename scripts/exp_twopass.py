"""Experiment: one-pass vs two-pass broadphase, single-thread vs split, per batch size.

    python scripts/exp_twopass.py
Verdicts of every variant must agree; prints the median kernel time (L2 flushed).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import ValidationContext, load_robot, runtime, workloads  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
import os  # noqa: E402
VARIANTS = {"x1": dict(split=False), "x1t": dict(split=False, two_pass=True),
            "x4": dict(split=True), "x4t": dict(split=True, two_pass=True),
            "dense": dict(split=False, early_exit=False), "dense4": dict(split=True, early_exit=False)}
if os.environ.get("VMP_EXP_SPLIT"):   # the forced split count applies to every variant
    VARIANTS = {"prod": dict(), "dense": dict(early_exit=False),
                "prod_np": dict(prune=False), "dense_np": dict(early_exit=False, prune=False)}


def timed(fn, reps=15):
    ts = []
    for r in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.mean(ts))   # event timer ticks are ~2 us: mean, not median


cases = [("cfg1", workloads.config1(1048576), n) for n in (4096, 16384, 65536, 131072, 262144)]
if not os.environ.get("VMP_EXP_CFG1_ONLY"):
    cases += [("cfg3", workloads.config3(), n) for n in (4096, 16384, 65536, 262144)]
    cases += [("cfg4", workloads.config4(), n) for n in (4096, 16384, 65536, 262144)]
for name, wl, n in cases:
    rob = load_robot(wl.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
    q = np.ascontiguousarray(wl.q[:, :n]) if wl.q.shape[1] >= n else np.ascontiguousarray(
        np.tile(wl.q, (1, -(-n // wl.q.shape[1])))[:, :n])
    qd = runtime.to_device(q)
    mod, denv = ctx.module, ctx.device_env
    ref = None
    row = []
    for tag, kw in VARIANTS.items():
        out = runtime.validate_device(mod, denv, qd, n, n, **kw)
        words = out.cpu().numpy()
        if ref is None:
            ref = words
        assert np.array_equal(words, ref), (name, n, tag)
        us = timed(lambda: runtime.validate_device(mod, denv, qd, n, n, out=out, **kw))
        row.append(f"{tag} {us:8.1f}")
    print(f"{name} n={n:8d}: " + "  ".join(row), flush=True)
