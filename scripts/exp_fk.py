"""FK-only kernel (vmp_fk_spheres) bandwidth: algorithmic bytes (joints in +
centres out) / kernel time, L2 flushed before each launch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import load_robot, runtime, workloads  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
for name in ("arm7", "fetch_standin", "baxter_standin"):
    rob = load_robot(name)
    n = 1 << 22
    q = torch.from_numpy(workloads.uniform_configs(rob.limits, n, 3)).cuda()
    rows = 3 * len(rob.program.checks)
    out = runtime.fk_spheres(rob.program, q)
    ts = []
    for r in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        runtime.fk_spheres(rob.program, q)
        b.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b) / 1e3)
    t = float(np.mean(ts))
    nbytes = n * 4 * (rob.program.dof + rows)
    print(f"{name}: {n} configs, {rows} rows: {t * 1e6:.1f} us, {nbytes / t / 1e9:.0f} GB/s "
          f"({nbytes / t / 1e9 / 6539.9:.3f} of 6540)", flush=True)

# write-only reference: torch fill of 1 GiB (what a pure store stream reaches here)
big = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
ts = []
for r in range(13):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    big.fill_(1.0)
    b.record()
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(a.elapsed_time(b) / 1e3)
t = float(np.mean(ts))
print(f"torch fill_ 1 GiB (write-only): {big.numel() * 4 / t / 1e9:.0f} GB/s")
