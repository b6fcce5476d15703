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

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

L2_FLUSH_BYTES = 256 << 20          # > 126 MB L2
PEAKS = ROOT / "MEASURED_PEAKS.json"
SMS = 148
FMA_PER_CLK = 128


# ----------------------------------------------------------------- helpers

def fp32_peak_tflops() -> tuple[float, str]:
    mhz = 1965.0
    src = "nominal sm_max_mhz 1965"
    if PEAKS.exists():
        mhz = float(json.loads(PEAKS.read_text()).get("sm_max_mhz", mhz))
        src = "MEASURED_PEAKS.json sm_max_mhz"
    return SMS * FMA_PER_CLK * 2 * mhz * 1e6 / 1e12, \
        f"148 SM x 128 FFMA/clk x 2 flop x {mhz:.0f} MHz ({src}); no tensor cores"


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
    peak, peak_src = fp32_peak_tflops()

    mw = workloads.config2()
    rob = load_robot(mw.robot)
    ctx = ValidationContext(rob.program, rob.model, rob.pairs, mw.env)
    E = len(mw.starts)
    # the public fixed-size API: resident edge buffers + CUDA graph of plan + rake
    mv = M.MotionValidator(ctx, E, mw.resolution, width=32)
    mv(mw.starts, mw.goals)
    torch.cuda.synchronize()
    sd, gd, bits = mv.starts, mv.goals, mv.bits
    mod, denv = ctx.module, ctx.device_env
    stream = torch.cuda.current_stream()

    def step():
        mv()                                              # one graph replay = one step

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
        step()
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
            step()
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
    achieved = flops_per_launch / (avg_launch_ms / 1e3) / 1e12

    # ---- end to end through the public API, host buffers: every step copies its
    # edges from pinned host memory and reads its verdict words back; the
    # 4-slot pipeline (a stream per slot) overlaps step k+1's H2D and rake with step k's drain
    hs = torch.from_numpy(mw.starts).pin_memory()
    hg = torch.from_numpy(mw.goals).pin_memory()
    depth = 4
    pipe = M.MotionPipeline(ctx, E, mw.resolution, width=32, depth=depth)
    for _ in range(args.warmup):
        pipe.result(pipe.submit(hs, hg))
    torch.cuda.synchronize()
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for st in pipe.streams:
        st.wait_event(a)
    inflight = []
    for i in range(args.steps):
        inflight.append(pipe.submit(hs, hg))
        if len(inflight) == depth:                        # oldest step's verdicts on the host
            got = pipe.result(inflight.pop(0))
    for t in inflight:
        got = pipe.result(t)
    pipe.wait_all(stream)
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b)
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = world * E / (e2e_ms / args.steps / 1e3)
    assert runtime.unpack_bits(got, E).tolist() == valid.tolist()

    fkcc = {} if args.no_aux else fkcc_summary(ctx_flush=flush, peak=peak)
    if rank != 0:
        return None
    line = {
        "metric": "validated edges/sec (raked motion validation, BASELINE config 2)",
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
        "config": {"workload": mw.name, "robot": "arm7 (Panda stand-in)", "edges_per_gpu": E,
                   "resolution": mw.resolution, "rake_width": 32,
                   "obstacles": "24 cuboids + 8 capsules",
                   "valid_edge_fraction": round(float(valid.mean()), 4),
                   "mean_states_per_edge": round(float(n_np.mean()), 2),
                   "l2": "flushed (256 MiB write) between timed steps; inputs 229 KB",
                   "launch": "CUDA graph (plan -> rake -> finalize, PDL edges) via motion.MotionValidator; "
                             "e2e through motion.MotionPipeline (4 slots, each step's H2D, "
                             "graph replay and D2H on its slot's own stream: step k+1's copy "
                             "and rake start while step k's rake drains)",
                   "parallelism": f"dp{world} (independent edges per rank)"},
        "roofline": {"bound": "fp32", "achieved": round(achieved, 3), "peak": round(peak, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                     "traffic": _traffic("vmp_motion_p1_s2_g1_o_ns"),
                     # the register-capped rake variant (loaded when it compiles
                     # without local memory; arm7: 96 registers, 5 CTAs / SM),
                     # built without sphere-obstacle code (config 2 has none)
                     "kernel": "vmp_motion_p1_s2_g1_o_ns",
                     "algorithmic_flop_per_state": f_state,
                     "states_counted_per_launch": int(states.sum()),
                     "note": "states fully evaluated by the rake (valid edges: all n; invalid: "
                             "iterations before the failing one) x reference dense flop/state; "
                             "peak: " + peak_src},
        # per step (one graph replay): cluster plan + rake + finalize kernels
        "gpu_launches": 3 * args.steps,
        "e2e": {"value": round(e2e_value, 1), "unit": "edges/s",
                "h2d_bytes_per_step": int(mw.starts.nbytes + mw.goals.nbytes),
                "d2h_bytes_per_step": int(bits.numel() * 4)},
        "clocks": clocks.summary(),
    }
    if fkcc:
        line["fkcc"] = fkcc
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_motion(mw, rob, processes=1, n_edges=args.cpu_edges)
    return line


def fkcc_summary(ctx_flush, peak: float) -> dict:
    """Configs 1/3/4 batch FK+CC: configs/s and % FP32 roofline (dense + early exit)."""
    import torch

    from paper_2309_14545_b200 import ValidationContext, codegen, load_robot, workloads
    from paper_2309_14545_b200 import runtime

    out = {}
    for key, make in (("cfg1", workloads.config1), ("cfg3", workloads.config3),
                      ("cfg4", workloads.config4)):
        wl = make()
        rob = load_robot(wl.robot)
        ctx = ValidationContext(rob.program, rob.model, rob.pairs, wl.env)
        n = wl.q.shape[1]
        f = codegen.algorithmic_flops(rob.program, rob.pairs, ctx.device_env.counts)["total"]
        res = {"robot": wl.robot, "configs": n, "flop_per_config": f}
        # product = the library's default kernel choice (early exit + broadphase,
        # or the straight-line dense kernel for sphere-only scenes); dense = every test
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
            words = cv.bits
            ms = float(np.mean(times))        # event ticks are ~2 us: mean of 20, not median
            rate = n / (ms / 1e3)
            res[mode] = {"ms": round(ms, 4), "configs_per_s": round(rate, 1),
                         "tflops": round(rate * f / 1e12, 3),
                         "frac_fp32": round(rate * f / 1e12 / peak, 4)}
        res["collision_rate"] = round(1 - float(runtime.unpack_bits(words.cpu().numpy(), n).mean()), 4)
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


# ------------------------------------------------------- CPU reference arm

_CPU = {}
# the reference package itself (pure Python / NumPy), staged git-ignored by
# scripts/run_reference_suite.sh --stage; it travels to the GPU box with the repo
REF_SRC = ROOT / "baseline" / "_ref" / "pkg" / "src"


def _ref_context(mw):
    """The reference's own ValidationContext(width=8) for config 2: its bundled
    arm7 URDF / sphere model compiled by its own tracing compiler, the scene
    converted to its primitive types.  None when the package is not staged."""
    if not (REF_SRC / "vecmp").is_dir():
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
    from paper_2309_14545_b200 import load_robot, workloads
    mw = workloads.config2()
    ref = _ref_context(mw)
    if ref is not None:
        _CPU.update(kind="reference", mw=mw, ctx=ref[0], rake=ref[1])
        return
    sys.path.insert(0, str(ROOT / "oracle"))
    import vecmp_oracle as O
    rob = load_robot(mw.robot)
    _CPU.update(kind="port", O=O, mw=mw, rob=rob, ob=O.Obstacles(mw.env.primitives))


def _cpu_worker(idx):
    if not _CPU:
        _cpu_init()
    mw = _CPU["mw"]
    if _CPU["kind"] == "reference":
        ctx, rake = _CPU["ctx"], _CPU["rake"]
        return [bool(rake(mw.starts[i], mw.goals[i], ctx, mw.resolution)) for i in idx]
    O, rob, ob = _CPU["O"], _CPU["rob"], _CPU["ob"]
    return [O.rake_check(rob.program, rob.pairs, ob, mw.starts[i], mw.goals[i], mw.resolution, 8)[0]
            for i in idx]


def _sample(n_edges: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(4096, size=min(n_edges, 4096), replace=False))


def cpu_baseline_motion(mw, rob, processes: int, n_edges: int) -> dict:
    """The reference (or, unstaged, its bit-exact oracle port) on one host
    core: the ValidationContext(width=8) rake per edge, as the reference runs it."""
    _cpu_init()
    idx = _sample(n_edges, 123)
    _cpu_worker(idx[:8])                                  # warm caches
    t0 = time.perf_counter()
    _cpu_worker(idx)
    wall = time.perf_counter() - t0
    what = "vecmp validate_motion_rake" if _CPU["kind"] == "reference" else "oracle port"
    return {"value": round(len(idx) / wall, 2), "unit": "edges/s", "cores": 1, "kind": _CPU["kind"],
            "sample": f"{len(idx)} seeded-random edges of the 4,096 ({what}, W=8 rake, numpy "
                      f"{np.__version__}, 1 process, {wall:.1f} s wall)"}


def run_reference(args, rank: int, world: int) -> dict | None:
    if rank != 0:
        return None
    import multiprocessing as mp

    from paper_2309_14545_b200 import load_robot, workloads
    mw = workloads.config2()
    rob = load_robot(mw.robot)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    per_step = max(cores * 8, 64)
    pool = mp.get_context("fork").Pool(cores, initializer=_cpu_init)
    try:
        for w in range(args.warmup):
            pool.map(_cpu_worker, np.array_split(_sample(cores, 7 + w), cores))
        t_total = 0.0
        for k in range(args.steps):
            idx = _sample(per_step, 1000 + k)
            t0 = time.perf_counter()
            pool.map(_cpu_worker, np.array_split(idx, cores))
            t_total += time.perf_counter() - t0
    finally:
        pool.close()
        pool.join()
    value = args.steps * per_step / t_total
    _cpu_init()                                           # this process: which arm ran
    kind = _CPU["kind"]
    what = "vecmp validate_motion_rake" if kind == "reference" else "oracle port of it"
    return {
        "impl": "reference",
        "metric": "validated edges/sec (raked motion validation, BASELINE config 2)",
        "value": round(value, 2), "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t_total / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; arm7 stand-in for Panda)",
        "config": {"workload": mw.name, "robot": "arm7 (Panda stand-in)", "resolution": mw.resolution,
                   "edges_per_step": per_step},
        "cpu_baseline": {"value": round(value, 2), "unit": "edges/s", "cores": cores, "kind": kind,
                         "sample": f"{per_step} seeded-random edges per step ({what}), W=8 "
                                   f"rake, one process per core"},
        "e2e": {"value": round(value, 2), "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


# -------------------------------------------------------------------- main

def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=("ours", "reference"))
    p.add_argument("--no-aux", action="store_true", help="skip the FK+CC batch summary")
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
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
