"""BASELINE config 5: Panda (arm7 stand-in) stress sweep on one B200.

Batch sizes 2^10 .. 2^24, environments of 16 / 128 / 1,024 mixed primitives
(50 % cuboids, 25 % capsules, 25 % spheres).  For every point: configs/s with
early exit + broadphase (product mode) and dense (every test), algorithmic
TFLOP/s and fraction of the FP32 peak (SURVEY.md §8d F = 487 + 220 P), and
the HBM traffic rate of the streamed batch.  Also times the FK-only kernel
(HBM-bound).  One JSON object per line.

Every point records the SM clock and throttle reasons sampled (nvidia-smi,
bench.ClockSampler) while its launches ran; fractions are of the FP32 peak
MEASURED on the same GPU (bench.measure_fp32_peak, first line).  Points with
N <= 2^18 are also timed "streamed": distinct resident batches (> 2x L2 in
total) validated by one graph of PDL-chained launches (ConfigStream).
"input_gbs" is algorithmic (4 dof + 1/8 byte per configuration / time), not
measured DRAM traffic; ncu DRAM bytes for selected points are in profiles/.

    python scripts/sweep_cfg5.py > profiles/round2_sweep_cfg5.jsonl
"""

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2309_14545_b200 import ValidationContext, codegen, load_robot, runtime, workloads  # noqa: E402


def timed(fn, reps=20, flush=None):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.mean(ts))          # event timestamps tick every 2.048 us: mean, not median


def main():
    torch.cuda.set_device(0)
    peaks = bench.measure_fp32_peak(0)
    peak = peaks["burst_tflops"]
    print(json.dumps({"fp32_peak": peaks}), flush=True)
    hbm = 6539.9
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    rob = load_robot("arm7")
    qall = torch.from_numpy(workloads.uniform_configs(rob.limits, 1 << 24, 50)).cuda()
    for p in (16, 128, 1024):
        env = workloads.config5_scene(p)
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, env)
        f = codegen.algorithmic_flops(rob.program, rob.pairs, ctx.device_env.counts)["total"]
        for lg in range(10, 25, 2):
            n = 1 << lg
            q = qall[:, :n]
            out = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
            row = {"P": p, "N": n, "flop_per_config": f}
            with bench.ClockSampler(0) as clk:
                for mode, early in (("product", True), ("dense", False)):
                    ms = timed(lambda: ctx.validate_batch(q, early_exit=early, out=out), flush=flush)
                    rate = n / (ms / 1e3)
                    row[mode] = {"ms": round(ms, 4), "configs_per_s": round(rate, 1),
                                 "alg_tflops": round(rate * f / 1e12, 2),
                                 "frac_fp32": round(rate * f / 1e12 / peak, 4),
                                 "input_gbs": round(rate * (7 * 4 + 1 / 8) / 1e9, 1)}
                if n <= (1 << 18):
                    copies = min(512, max(4, -(-2 * (126 << 20) // (7 * 4 * n))))
                    cs = ctx.stream_validator(n, copies)
                    for i in range(copies):
                        cs.load(i, q)
                    ms = timed(cs, reps=5, flush=flush) / copies
                    rate = n / (ms / 1e3)
                    row["streamed"] = {"ms": round(ms, 4), "configs_per_s": round(rate, 1),
                                       "alg_tflops": round(rate * f / 1e12, 2),
                                       "frac_fp32": round(rate * f / 1e12 / peak, 4),
                                       "batches": copies}
                    del cs
                time.sleep(0.25)          # let the sampler see this point's load
            row["clocks"] = clk.summary()
            if lg == 20:
                v = runtime.unpack_bits(out.cpu().numpy(), n)
                row["collision_rate"] = round(1 - float(v.mean()), 4)
            print(json.dumps(row), flush=True)
    # FK-only kernel: HBM bound
    for name in ("arm7", "fetch_standin", "baxter_standin"):
        r = load_robot(name)
        q = torch.from_numpy(workloads.uniform_configs(r.limits, 1 << 22, 60)).cuda()
        n = q.shape[1]
        outb = torch.empty((3 * len(r.program.checks), n), dtype=torch.float32, device="cuda")
        mod = runtime.robot_module(r.program)

        def fk():
            runtime.check(runtime.lib().vmp_fk_spheres(mod.handle, q.data_ptr(), n, n,
                                                       outb.data_ptr(), n, runtime.stream_handle()))
        ms = timed(fk, flush=flush)
        nbytes = n * (4 * r.program.dof + 12 * len(r.program.checks))
        print(json.dumps({"kernel": "vmp_fk_spheres", "robot": name, "N": n, "ms": round(ms, 4),
                          "bytes": nbytes, "gbs": round(nbytes / (ms / 1e3) / 1e9, 1),
                          "frac_hbm": round(nbytes / (ms / 1e3) / 1e9 / hbm, 4)}), flush=True)


if __name__ == "__main__":
    main()
