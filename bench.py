"""Benchmark: raked motion validation (BASELINE config 2) on B200, one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg1|cfg3|cfg4|cfg5_<P>_<log2N>]

Headline (default): BASELINE.json config 2 - 4,096 arm7 ("Panda" stand-in)
edges, resolution 1/32, 24 cuboids + 8 capsules; one step = validate every
edge (one kernel launch).  ``value`` = edges/s over all ranks with inputs
resident in HBM; ``e2e`` = the same through the public API with the edges
copied from pinned host memory and the verdict bits read back every step.
The FK+CC batch workloads (configs 1, 3, 4) are reported alongside under
``fkcc`` (configs/s and % of the FP32 roofline).

Multi-GPU: one process per GPU (torchrun), every rank validates its own
4,096-edge batch (weak scaling, no data-path collective - the path shards
into independent edges); time = max over ranks.

``--impl reference`` times the reference on the host CPU cores: the
reference package itself (vecmp's own validate_motion_rake, tracing compiler
and bundled arm7, W = 8 blocks) when it is staged under baseline/_ref/pkg,
else its bit-exact oracle port (oracle/vecmp_oracle.py); one process per
core, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

L2_FLUSH_BYTES = 256 << 20          # > 126 MB L2
PEAKS = ROOT / "MEASURED_PEAKS.json"
SMS = 148
FMA_PER_CLK = 128


# ----------------------------------------------------------------- helpers

def nominal_fp32_tflops() -> float:
    mhz = 1965.0
    if PEAKS.exists():
        mhz = float(json.loads(PEAKS.read_text()).get("sm_max_mhz", mhz))
    return SMS * FMA_PER_CLK * 2 * mhz * 1e6 / 1e12


def measure_fp32_peak(device: int) -> dict:
    """Measured FP32 FMA-pipe peak on this GPU (vmp_bench_ffma: 4 independent
    FFMA chains per thread, 64 warps per SM).  ``burst``: best of 5 single
    ~3 ms launches (the regime of a kernel timed alone - the bench steps are
    tens of us with an L2 flush between them); ``sustained``: ~2 s of
    back-to-back launches, with the SM clock sampled meanwhile."""
    import ctypes

    from paper_2309_14545_b200._native import check, lib
    iters = 1500

    def run(launches: int) -> float:
        t, ms = ctypes.c_double(), ctypes.c_double()
        check(lib().vmp_bench_ffma(iters, launches, ctypes.byref(t), ctypes.byref(ms)))
        return t.value

    run(1)
    burst = max(run(1) for _ in range(5))
    with ClockSampler(device) as clk:
        sustained = run(600)
    return {"burst_tflops": round(burst, 2), "sustained_tflops": round(sustained, 2),
            "nominal_tflops": round(nominal_fp32_tflops(), 2),
            "sustained_clocks": clk.summary(),
            "kernel": "vmp_k_ffma (libvmp vmp_bench_ffma)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._drain, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _drain(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[2:]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def rake_state_counts(n: np.ndarray, blocks: np.ndarray, valid: np.ndarray, width: int = 32):
    """States the rake must fully evaluate: all n for valid edges; for invalid
    edges the in-range states of the iterations before the failing one."""
    s = np.ceil(n / width).astype(np.int64)
    full = n.copy()
    done = np.where(valid, blocks, blocks - 1)            # completed iterations
    # in-range states of iterations 1..d: sum_k min(max(n - k s, 0), d)
    k = np.arange(width)[None, :]
    per = np.clip(n[:, None] - k * s[:, None], 0, None)
    part = np.minimum(per, done[:, None]).sum(axis=1)
    return np.where(valid, full, part)


def _traffic(kernel: str):
    """DRAM bytes per launch of ``kernel`` from the committed ncu capture, or None."""
    path = ROOT / "profiles" / "traffic.json"
    if not path.exists():
        return None
    return json.loads(path.read_text()).get(kernel)




def _executed(kernel: str):
    """Executed FP32 flop per launch of ``kernel`` (ncu SASS op counts,
    profiles/executed.json), or None."""
    path = ROOT / "profiles" / "executed.json"
    if not path.exists():
        return None
    return json.loads(path.read_text()).get(kernel)


PARITY = ROOT / "tests" / "golden" / "bench_parity.npz"
E2E_REPS = 5


def _bits(words, n: int) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(words).astype(np.uint32, copy=False))
    return np.unpackbits(w.view(np.uint8), bitorder="little")[:n].astype(bool)


def batch_parity(key: str, words) -> dict | None:
    """Our verdicts of a full bench batch vs the reference's (fixture written by
    tests/golden/make_bench_parity.py from the bit-exact oracle): mismatches
    outside the +-1e-4 m clearance band must be 0; in-band ones are counted."""
    if not PARITY.exists():
        return None
    fx = np.load(PARITY)
    n = int(fx[f"{key}_n"])
    got, ref = _bits(words, n), _bits(fx[f"{key}_ref_words"], n)
    band = np.zeros(n, bool)
    band[fx[f"{key}_band_idx"]] = True
    diff = got != ref
    return {"configs": n, "band": int(band.sum()), "band_mismatches": int((diff & band).sum()),
            "mismatches_outside_band": int((diff & ~band).sum())}


def motion_parity(valid: np.ndarray) -> dict | None:
    if not PARITY.exists():
        return None
    fx = np.load(PARITY)
    ref = fx["cfg2_ref_verdict"]
    crit = fx["cfg2_band_critical"]
    return {"edges": int(len(ref)), "mismatches": int((valid != ref).sum()),
            "band_states": int(fx["cfg2_band_states"].sum()),
            "band_critical_edges": [int(e) for e in crit],
            "band_critical_mismatches": int((valid[crit] != ref[crit]).sum())}


CFG2_CONFIG = {"workload": "cfg2_arm7_4096edges_24box_8cap", "robot": "arm7 (Panda stand-in)",
               "edges_per_gpu": 4096, "resolution": 1.0 / 32.0,
               "obstacles": "24 cuboids + 8 capsules (keep-out 0.3 m)",
               "edges": "seeded, even-indexed edges forced collision-free "
                        "(paper_2309_14545_b200/data/cfg2_edges.npz)"}
METRIC = "validated edges/sec (raked motion validation, BASELINE config 2)"


# ----------------------------------------------------------- our GPU arm

def run_ours(args, rank: int, world: int) -> dict | None:
    import torch
    import torch.distributed as dist

    from paper_2309_14545_b200 import ValidationContext, codegen, load_robot, workloads
    from paper_2309_14545_b200 import motion as M
    from paper_2309_14545_b200 import runtime

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    mw = workloads.config2()
    rob = load_robot(mw.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
    E = len(mw.starts)
    # the public fixed-size API: resident edge buffers + CUDA graph of begin + rake
    mv = M.MotionValidator(ctx, E, mw.resolution, width=32)
    mv(mw.starts, mw.goals)
    torch.cuda.synchronize()
    sd, gd, bits = mv.starts, mv.goals, mv.bits
    mod, denv = ctx.module, ctx.device_env
    stream = torch.cuda.current_stream()

    # the roofline denominator, measured on this GPU (VMP_BENCH_PEAK_FIRST=1: before
    # the timed regions instead of after them - an experiment switch)
    peak_first = os.environ.get("VMP_BENCH_PEAK_FIRST") == "1"
    peaks = measure_fp32_peak(dev) if peak_first else None

    # per-edge counts for the roofline numerator (one extra untimed launch)
    b0, ns_t, bl_t = runtime.validate_motions_device(mod, denv, sd, gd, mw.resolution, width=32,
                                                     prune=True, want_counts=True)
    valid = runtime.unpack_bits(b0.cpu().numpy(), E)
    n_np, b_np = ns_t.cpu().numpy().astype(np.int64), bl_t.cpu().numpy().astype(np.int64)
    states = rake_state_counts(n_np, b_np, valid)
    f_cfg = codegen.algorithmic_flops(rob.program, rob.pairs, denv.counts)["total"]
    f_state = f_cfg + 3 * rob.program.dof                    # + interpolation
    flops_per_launch = float(states.sum()) * f_state

    for _ in range(args.warmup):
        mv()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        for a, b in ev:
            flush.zero_()                                 # L2 flush between timed steps
            a.record(stream)
            mv()                                          # one step = one graph replay
            b.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    kernel_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(kernel_ms))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * E / (ms_per_step / 1e3)
    avg_launch_ms = float(np.mean(kernel_ms))
    got_valid = runtime.unpack_bits(mv.host_bits(), E)

    # ---- end to end through the public API, host buffers: every step copies its
    # edges from pinned host memory and reads its verdict words back; the
    # 4-slot pipeline (a stream per slot) overlaps step k+1's H2D and rake with step k's drain
    hs = torch.from_numpy(mw.starts).pin_memory()
    hg = torch.from_numpy(mw.goals).pin_memory()
    depth = 6
    pipe = M.MotionPipeline(ctx, E, mw.resolution, width=32, depth=depth)
    for _ in range(max(args.warmup, depth)):              # every slot has run once
        pipe.result(pipe.submit(hs, hg))
    # the K-step region lasts under a millisecond, so one host hiccup moves it by
    # tens of percent: it is timed E2E_REPS times, each from an empty pipeline to
    # an empty one, and the median is reported (every repetition is in e2e.runs)
    e2e_runs = []
    for _ in range(E2E_REPS):
        torch.cuda.synchronize()
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for st in pipe.streams:
            st.wait_event(a)
        inflight = []
        for i in range(args.steps):
            inflight.append(pipe.submit(hs, hg))
            if len(inflight) == depth:                    # oldest step's verdicts on the host
                got = pipe.result(inflight.pop(0))
        for t in inflight:
            got = pipe.result(t)
        pipe.wait_all(stream)
        b.record(stream)
        torch.cuda.synchronize()
        e2e_runs.append(a.elapsed_time(b))
    e2e_ms = float(np.median(e2e_runs))
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = world * E / (e2e_ms / args.steps / 1e3)
    assert runtime.unpack_bits(got, E).tolist() == valid.tolist()
    assert got_valid.tolist() == valid.tolist()

    if peaks is None:
        peaks = measure_fp32_peak(dev)
    peak = peaks["burst_tflops"]
    achieved = flops_per_launch / (avg_launch_ms / 1e3) / 1e12
    if rank != 0:
        return None
    aux = not args.no_aux
    fkcc = fkcc_summary(ctx_flush=flush, peak=peak) if aux else {}
    executed = _executed("vmp_motion_p1_s2_g1_o_ns")
    roofline = {"bound": "fp32", "achieved": round(achieved, 3), "peak": peak,
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                "traffic": _traffic("vmp_motion_p1_s2_g1_o_ns"),
                # the register-capped rake variant (loaded when it compiles
                # without local memory; arm7: 96 registers, 5 CTAs / SM),
                # built without sphere-obstacle code (config 2 has none)
                "kernel": "vmp_motion_p1_s2_g1_o_ns",
                "algorithmic_flop_per_state": f_state,
                "states_counted_per_launch": int(states.sum()),
                "peak_measured": peaks,
                "note": "achieved = states the rake must fully evaluate (valid edges: all n; "
                        "invalid: the iterations before the failing one) x the reference's "
                        "dense flop per state / mean step time (begin + rake + finalize); a fraction above 1 is work the exact broadphase avoided, executed_frac is what ran; "
                        "peak = measured FFMA burst (peak_measured); no tensor cores"}
    if executed:
        ex = float(executed["flop_per_launch"])
        roofline["executed_frac"] = round(ex / (avg_launch_ms / 1e3) / 1e12 / peak, 4)
        roofline["executed_flop_per_launch"] = ex
        roofline["executed_source"] = executed.get("source", "profiles/executed.json")
    line = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "edges/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded; arm7 stand-in for Panda, see DESIGN.md)",
        "config": dict(CFG2_CONFIG),
        "setup": {"rake_width": 32, "parallelism": f"dp{world} (independent edges per rank)",
                  "valid_edge_fraction": round(float(valid.mean()), 4),
                  "mean_states_per_edge": round(float(n_np.mean()), 2),
                  "l2": "flushed (256 MiB write) between timed steps; inputs 229 KB",
                  "launch": "CUDA graph (begin -> dynamic-queue rake -> finalize, PDL edges) via "
                            "motion.MotionValidator; e2e through motion.MotionPipeline (6 slots, "
                            "each step's H2D, graph replay and D2H on its slot's own stream)"},
        "roofline": roofline,
        # per step (one graph replay): begin + rake + finalize kernels
        "gpu_launches": 3 * args.steps,
        "e2e": {"value": round(e2e_value, 1), "unit": "edges/s",
                "runs_ms": [round(x, 4) for x in e2e_runs],
                "note": f"median of {E2E_REPS} repetitions of the {args.steps}-step region",
                "h2d_bytes_per_step": int(mw.starts.nbytes + mw.goals.nbytes),
                "d2h_bytes_per_step": int(bits.numel() * 4)},
        "clocks": clocks.summary(),
        "parity": {"cfg2": motion_parity(valid)},
    }
    if fkcc:
        for key in ("cfg1", "cfg3", "cfg4"):
            line["parity"][key] = fkcc[key].pop("parity")
        line["fkcc"] = fkcc
        line["latency"] = latency_summary(mw, rob)
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"], line["cpu_baselines"] = cpu_baselines(args.cpu_edges)
        if "latency" in line:
            line["latency"]["reference"] = line["cpu_baselines"].pop("latency", None)
    return line


def fkcc_summary(ctx_flush, peak: float) -> dict:
    """Configs 1/3/4 batch FK+CC: configs/s and % of the measured FP32 peak
    (product mode = the library's kernel choice; dense = every test), plus
    verdict parity of the full batch against the reference's verdicts."""
    import torch

    from paper_2309_14545_b200 import ValidationContext, codegen, load_robot, workloads

    out = {}
    for key, make in (("cfg1", workloads.config1), ("cfg3", workloads.config3),
                      ("cfg4", workloads.config4)):
        wl = make()
        rob = load_robot(wl.robot)
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
        n = wl.q.shape[1]
        f = codegen.algorithmic_flops(rob.program, rob.pairs, ctx.device_env.counts)["total"]
        res = {"robot": wl.robot, "configs": n, "flop_per_config": f}
        words = {}
        for mode, early in (("product", True), ("dense", False)):
            cv = ctx.batch_validator(n, early_exit=early)       # resident batch + CUDA graph
            cv(wl.q)
            for _ in range(3):
                cv()
            times = []
            for _ in range(20):
                ctx_flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                cv()
                b.record()
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
            words[mode] = cv.bits.cpu().numpy()
            ms = float(np.mean(times))        # event ticks are ~2 us: mean of 20, not median
            rate = n / (ms / 1e3)
            res[mode] = {"ms": round(ms, 4), "configs_per_s": round(rate, 1),
                         "tflops": round(rate * f / 1e12, 3),
                         "frac_fp32": round(rate * f / 1e12 / peak, 4)}
            ex = _executed(f"{key}_{mode}")
            if ex:
                res[mode]["executed_frac"] = round(ex["flop_per_launch"] / (ms / 1e3) / 1e12 / peak, 4)
        # streamed: `copies` resident batches (together > 2x L2, so every batch reads
        # its configurations from HBM) validated by one graph of PDL-chained launches;
        # the L2 is flushed before each replay; per batch = replay time / copies
        copies = max(4, -(-2 * (126 << 20) // wl.q.nbytes))
        cs = ctx.stream_validator(n, copies)
        for i in range(copies):
            cs.load(i, wl.q)
        cs()
        times = []
        for _ in range(5):
            ctx_flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            cs()
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b) / copies)
        ms = float(np.mean(times))
        rate = n / (ms / 1e3)
        res["streamed"] = {"ms": round(ms, 4), "configs_per_s": round(rate, 1),
                           "tflops": round(rate * f / 1e12, 3),
                           "frac_fp32": round(rate * f / 1e12 / peak, 4), "batches": copies,
                           "note": "product kernels, one graph of PDL-chained launches over "
                                   "distinct resident batches (total > 2x L2), L2 flushed "
                                   "before the graph; ms per batch"}
        for i in range(copies):
            assert np.array_equal(cs.bits[i].cpu().numpy(), words["product"])
        del cs
        assert np.array_equal(words["product"], words["dense"])
        res["collision_rate"] = round(1 - float(_bits(words["product"], n).mean()), 4)
        res["parity"] = batch_parity(key, words["product"])
        out[key] = res
    out["fk_only"] = fk_only_summary(ctx_flush)
    return out


def fk_only_summary(ctx_flush, n: int = 1 << 22) -> dict:
    """FK-only kernel (vmp_fk_spheres): the HBM-bound row.
    Algorithmic bytes = joints in (4 dof) + centres out (12 per marker) per
    configuration; peak = MEASURED_PEAKS.json hbm_gbs (copy bandwidth)."""
    import torch

    from paper_2309_14545_b200 import load_robot, runtime, workloads

    hbm = float(json.loads(PEAKS.read_text()).get("hbm_gbs", 6540.0)) if PEAKS.exists() else 6540.0
    out = {"configs": n, "peak_gbs": hbm}
    for name in ("arm7", "baxter_standin"):
        rob = load_robot(name)
        q = torch.from_numpy(workloads.uniform_configs(rob.limits, n, 3)).cuda()
        rows = 3 * len(rob.program.checks)
        runtime.fk_spheres(rob.program, q)
        times = []
        for _ in range(10):
            ctx_flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            runtime.fk_spheres(rob.program, q)
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b) / 1e3)
        t = float(np.mean(times))
        gbs = n * 4 * (rob.program.dof + rows) / t / 1e9
        out[name] = {"bytes_per_config": 4 * (rob.program.dof + rows), "us": round(t * 1e6, 1),
                     "gbs": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4)}
    return out


def latency_summary(mw, rob, calls: int = 300) -> dict:
    """Per-call latency of the reference-signature single-request API (what
    the reference's planners call one at a time, planners.py:119-123,152-168,
    simplify.py:82-86): state_valid and a W = 8 validate_block
    (ValidationContext(width=8)), and a single-edge raked_motion_check - host
    inputs and results, one synchronising C call each (vmp_*_host).  Host
    wall clock per call (the GPU work is synchronous inside the call)."""
    from paper_2309_14545_b200 import ConfigBlock, ValidationContext
    from paper_2309_14545_b200 import motion as M

    ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env, width=8)
    q = np.ascontiguousarray(mw.starts[:8].T)
    block = ConfigBlock(dim=q.shape[0], width=8, data=q, valid_count=8)

    def per_call(fn, n):
        for _ in range(20):
            fn(0)
        t0 = time.perf_counter()
        for i in range(n):
            fn(i)
        return round((time.perf_counter() - t0) / n * 1e6, 2)

    return {
        "state_valid_us": per_call(lambda i: ctx.state_valid(mw.starts[i % 4096]), calls),
        "validate_block_w8_us": per_call(lambda i: ctx.validate_block(block), calls),
        "raked_motion_check_us": per_call(
            lambda i: M.raked_motion_check(mw.starts[i % 4096], mw.goals[i % 4096], ctx,
                                           mw.resolution), calls),
        "note": "ValidationContext(width=8); raked_motion_check averaged over the first "
                f"{calls} config-2 edges (begin + rake + finalize per call)",
    }


# ------------------------------------------------------- CPU reference arm

_CPU = {}
# the reference package itself (pure Python / NumPy), git-ignored, travels to the
# GPU box with the repo: the offline pip install into baseline/_ref (DESIGN.md
# §5), else the source tree staged by scripts/run_reference_suite.sh --stage
REF_SRC = next((d for d in (ROOT / "baseline" / "_ref", ROOT / "baseline" / "_ref" / "pkg" / "src")
                if (d / "vecmp" / "collision.py").is_file()), ROOT / "baseline" / "_ref")


def _ref_context(mw):
    """The reference's own ValidationContext(width=8) for config 2: its bundled
    arm7 URDF / sphere model compiled by its own tracing compiler, the scene
    converted to its primitive types.  None when the package is not staged."""
    if not (REF_SRC / "vecmp" / "collision.py").is_file():
        return None
    sys.path.insert(0, str(REF_SRC))
    import vecmp.collision as RC
    from vecmp.motion import validate_motion_rake
    from vecmp.planners import build_robot
    from vecmp.resources import robot_path
    from vecmp.robot import load_sphere_model, parse_urdf
    tree = parse_urdf(robot_path("arm7.urdf").read_text())
    rob = build_robot(tree, load_sphere_model(tree, robot_path("arm7_spheres.yaml").read_text()))
    prims = []
    for p in mw.env.primitives:
        if hasattr(p, "p0"):
            prims.append(RC.CapsuleObstacle(p0=np.asarray(p.p0, float), p1=np.asarray(p.p1, float),
                                            radius=float(p.radius)))
        elif hasattr(p, "half_extents"):
            prims.append(RC.BoxObstacle(center=np.asarray(p.center, float),
                                        half_extents=np.asarray(p.half_extents, float),
                                        rotation=np.asarray(p.rotation, float)))
        else:
            prims.append(RC.SphereObstacle(center=np.asarray(p.center, float),
                                           radius=float(p.radius)))
    env = RC.Environment(primitives=prims, name=mw.env.name)
    ctx = RC.ValidationContext(program=rob.program, model=rob.model, pairs=rob.pairs, env=env,
                               width=8)
    return ctx, validate_motion_rake


def _cpu_init() -> None:
    """Per-process state of the CPU arm: the reference package when staged
    (kind "reference"), else the oracle port (kind "port"); workload."""
    if _CPU:
        return
    from paper_2309_14545_b200 import load_robot, workloads
    mw = workloads.config2()
    ref = _ref_context(mw)
    sys.path.insert(0, str(ROOT / "oracle"))
    import vecmp_oracle as O
    _CPU.update(O=O, mw=mw)
    if ref is not None:
        _CPU.update(kind="reference", ctx=ref[0], rake=ref[1])
        return
    rob = load_robot(mw.robot)
    _CPU.update(kind="port", rob=rob, ob=O.Obstacles(mw.env.primitives))


def _cpu_worker(idx):
    """Config-2 edges ``idx`` through the W = 8 rake, as the reference runs it."""
    _cpu_init()
    mw = _CPU["mw"]
    if _CPU["kind"] == "reference":
        ctx, rake = _CPU["ctx"], _CPU["rake"]
        return [bool(rake(mw.starts[i], mw.goals[i], ctx, mw.resolution)) for i in idx]
    O, rob, ob = _CPU["O"], _CPU["rob"], _CPU["ob"]
    return [O.rake_check(rob.program, rob.pairs, ob, mw.starts[i], mw.goals[i], mw.resolution, 8)[0]
            for i in idx]


_FKCC = {}


def _fkcc_workload(key: str):
    if key not in _FKCC:
        from paper_2309_14545_b200 import load_robot, workloads
        wl = {"cfg1": workloads.config1, "cfg3": workloads.config3, "cfg4": workloads.config4}[key]()
        rob = load_robot(wl.robot)
        _FKCC[key] = (wl, rob, _CPU["O"].Obstacles(wl.env.primitives))
    return _FKCC[key]


def _fkcc_job(job):
    """FK+CC on the CPU (oracle port of the reference's validate_block, prune on
    as ValidationContext's default): ``asis`` = W = 8 blocks, the reference's
    own width; ``wide`` = one block over the whole slice."""
    _cpu_init()
    key, mode, lo, hi = job
    O = _CPU["O"]
    wl, rob, ob = _fkcc_workload(key)
    q = wl.q[:, lo:hi]
    t0 = time.perf_counter()
    if mode == "asis":
        for i in range(0, q.shape[1], 8):
            O.validate_lanes(rob.program, rob.pairs, ob, np.ascontiguousarray(q[:, i:i + 8]))
    else:
        O.validate_lanes(rob.program, rob.pairs, ob, np.ascontiguousarray(q))
    return key, mode, hi - lo, time.perf_counter() - t0


def _motion_job(job):
    _cpu_init()
    t0 = time.perf_counter()
    _cpu_worker(job[1])
    return "cfg2", "asis", len(job[1]), time.perf_counter() - t0


def _latency_job(_):
    """Per-call latency of the reference API on one core: state_valid and one
    W = 8 validate_block (oracle port of validate_block), and one W = 8 rake."""
    _cpu_init()
    O, mw = _CPU["O"], _CPU["mw"]
    from paper_2309_14545_b200 import load_robot
    rob = load_robot(mw.robot)
    ob = O.Obstacles(mw.env.primitives)
    q8 = np.ascontiguousarray(mw.starts[:8].T)
    t0 = time.perf_counter()
    for i in range(200):
        O.validate_lanes(rob.program, rob.pairs, ob, np.repeat(mw.starts[i][:, None], 8, axis=1))
    sv = (time.perf_counter() - t0) / 200
    t0 = time.perf_counter()
    for _ in range(200):
        O.validate_lanes(rob.program, rob.pairs, ob, q8)
    vb = (time.perf_counter() - t0) / 200
    t0 = time.perf_counter()
    for i in range(100):
        O.rake_check(rob.program, rob.pairs, ob, mw.starts[i], mw.goals[i], mw.resolution, 8)
    rk = (time.perf_counter() - t0) / 100
    return {"state_valid_us": round(sv * 1e6, 1), "validate_block_w8_us": round(vb * 1e6, 1),
            "raked_motion_check_us": round(rk * 1e6, 1),
            "kind": "port", "note": "oracle port of the reference API on 1 host core; "
                                    "rake averaged over the first 100 config-2 edges"}


def _cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def _cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _sample(n_edges: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(4096, size=min(n_edges, 4096), replace=False))


def cpu_baselines(motion_edges: int, prefix: int = 65536) -> tuple[dict, dict]:
    """The reference CPU path on this box's host cores:

    * config 2 motion: ``motion_edges`` seeded edges through the W = 8 rake on
      one core (the headline ``cpu_baseline``);
    * configs 1 / 3 / 4 FK+CC: (1) as-is - W = 8 validate_block blocks on a
      ``prefix``-configuration prefix, one core; (2) wide - the same prefix as
      one block, one core; (3) wide x cores - the whole batch split over every
      core, one process each;
    * per-call latency of the reference API (one core).

    Phase 1 runs the single-core jobs concurrently, one process per job;
    phase 2 the all-core runs.  The oracle port is bit-exact to the reference
    (tests/test_oracle_golden.py); the reference package itself is used for
    the motion job when staged under baseline/_ref/pkg."""
    import multiprocessing as mp

    cores = _cores()
    _cpu_init()
    kind = _CPU["kind"]
    mctx = mp.get_context("fork")
    idx = _sample(motion_edges, 123)
    jobs = [("cfg2", idx)] + [(k, m, 0, prefix) for k in ("cfg1", "cfg3", "cfg4")
                              for m in ("asis", "wide")]
    t_start = time.perf_counter()
    with mctx.Pool(min(cores, len(jobs) + 1)) as pool:
        lat = pool.apply_async(_latency_job, (0,))
        res = pool.map(lambda_dispatch, jobs, chunksize=1)
        latency = lat.get()
    rates = {(k, m): n / t for k, m, n, t in res}
    wide_all = {}
    with mctx.Pool(cores) as pool:
        for key in ("cfg1", "cfg3", "cfg4"):
            n = {"cfg1": 65536, "cfg3": 1 << 20, "cfg4": 1 << 20}[key]
            bounds = np.linspace(0, n, cores + 1).astype(int)
            pool.map(_fkcc_job, [(key, "wide", 0, 64)] * cores)          # warm every worker
            t0 = time.perf_counter()
            pool.map(_fkcc_job, [(key, "wide", lo, hi) for lo, hi in zip(bounds, bounds[1:])],
                     chunksize=1)
            wide_all[key] = n / (time.perf_counter() - t0)
    wall = time.perf_counter() - t_start
    what = "vecmp validate_motion_rake" if kind == "reference" else "oracle port"
    motion = {"value": round(rates[("cfg2", "asis")], 2), "unit": "edges/s", "cores": 1,
              "kind": kind,
              "sample": f"{len(idx)} seeded-random edges of the 4,096 ({what}, W=8 rake, numpy "
                        f"{np.__version__}, 1 process)"}
    fk = {"host": {"cores": cores, "cpu_model": _cpu_model(), "numpy": np.__version__,
                   "wall_s": round(wall, 1)},
          "latency": latency}
    for key in ("cfg1", "cfg3", "cfg4"):
        fk[key] = {"unit": "configs/s", "kind": "port",
                   "asis_w8_1core": round(rates[(key, "asis")], 1),
                   "wide_1core": round(rates[(key, "wide")], 1),
                   "wide_all_cores": round(wide_all[key], 1),
                   "sample": f"as-is / wide: first {prefix} configurations of the batch "
                             f"(W=8 blocks / one block, 1 core); wide x cores: the whole "
                             f"batch, one process per core ({cores})"}
    return motion, fk


def lambda_dispatch(job):
    return _motion_job(job) if job[0] == "cfg2" else _fkcc_job(job)


def run_reference(args, rank: int, world: int) -> dict | None:
    """The reference CPU path on this box's host cores, every step validating
    the FULL 4,096-edge config-2 batch (W = 8 rake per edge, one process per
    core, edges dealt round-robin in chunks)."""
    if rank != 0:
        return None
    import multiprocessing as mp

    cores = _cores()
    E = 4096
    chunks = [np.arange(i, E, cores * 4) for i in range(cores * 4)]   # balanced, interleaved
    pool = mp.get_context("fork").Pool(cores, initializer=_cpu_init)
    try:
        for w in range(args.warmup):
            pool.map(_cpu_worker, [c[:1] for c in chunks[:cores]])
        t_total = 0.0
        verdicts = None
        for k in range(args.steps):
            t0 = time.perf_counter()
            parts = pool.map(_cpu_worker, chunks, chunksize=1)
            t_total += time.perf_counter() - t0
            if verdicts is None:
                verdicts = np.zeros(E, bool)
                for c, v in zip(chunks, parts):
                    verdicts[c] = v
    finally:
        pool.close()
        pool.join()
    value = args.steps * E / t_total
    _cpu_init()                                           # this process: which arm ran
    kind = _CPU["kind"]
    what = "vecmp validate_motion_rake" if kind == "reference" else "oracle port of it"
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 2), "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t_total / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; arm7 stand-in for Panda, see DESIGN.md)",
        "config": dict(CFG2_CONFIG),
        "setup": {"rake_width": 8, "parallelism": f"{cores} host processes (one per core)",
                  "valid_edge_fraction": round(float(verdicts.mean()), 4)},
        "cpu_baseline": {"value": round(value, 2), "unit": "edges/s", "cores": cores, "kind": kind,
                         "sample": f"every step the full {E}-edge batch ({what}, W=8 rake), "
                                   f"one process per core, {_cpu_model()}"},
        "e2e": {"value": round(value, 2), "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "parity": {"cfg2": motion_parity(verdicts)},
    }


# -------------------------------------------------------------------- main

def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=("ours", "reference"))
    p.add_argument("--no-aux", action="store_true",
                   help="skip the FK+CC batch summary, parity and latency sections")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-edges", type=int, default=1024)
    args = p.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    line = run_ours(args, rank, world) if args.impl == "ours" else run_reference(args, rank, world)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
