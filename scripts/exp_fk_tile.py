"""Experiment: vmp_fk_spheres tile size (configurations per thread) vs bandwidth.

    python scripts/exp_fk_tile.py 1,2,4
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from exp_variants import module_for  # noqa: E402
from paper_2309_14545_b200 import codegen, load_robot, runtime, workloads  # noqa: E402
from paper_2309_14545_b200._native import check, lib  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
for per in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4").split(",")]:
    codegen.FK_SMEM_TILE = 224 * 1024
    codegen.fk_tiling = lambda rows, p=per: (p, 2 if 2 * rows * 128 * p * 4 <= 80 * 1024 else 1)
    for name in ("arm7", "fetch_standin", "baxter_standin"):
        rob = load_robot(name)
        try:
            mod = module_for(rob, 0)
        except RuntimeError as exc:                    # tile does not fit in shared memory
            print(f"per_thread={per} {name}: skipped ({exc})", flush=True)
            continue
        n = 1 << 22
        q = torch.from_numpy(workloads.uniform_configs(rob.limits, n, 3)).cuda()
        rows = 3 * len(rob.program.checks)
        out = torch.empty((rows, n), dtype=torch.float32, device="cuda")

        def run():
            check(lib().vmp_fk_spheres(mod.handle, q.data_ptr(), n, n, out.data_ptr(), n,
                                       runtime.stream_handle()))
        run()
        ref = runtime.fk_spheres(rob.program, q)
        assert torch.equal(ref, out), (per, name)
        ts = []
        for r in range(13):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run()
            b.record()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(a.elapsed_time(b) / 1e3)
        t = float(np.mean(ts))
        nbytes = n * 4 * (rob.program.dof + rows)
        print(f"per_thread={per} {name}: {t * 1e6:.1f} us, {nbytes / t / 1e9:.0f} GB/s", flush=True)
