"""Straight-line motion validation with the stratified rake, on the B200.

Reference semantics (pkg/src/vecmp/motion.py): a motion is discretised into
n = max(1, ceil(||g - s|| / resolution)) states at t = i/n, i = 1..n (goal
checked, start not); with W lanes and s = ceil(n / W), lane k owns indices
k*s + j, j = 1..s, iteration j checks one index per stratum and the rake
stops at the first iteration containing an invalid in-range state.

Device design (csrc/vmp_device.cuh, codegen.py ``vmp_motion_*``): one warp
per edge taken from a persistent atomic queue; the warp walks the W-rake's
state sequence 32 states at a time (for W = 32 exactly one rake iteration
per step), interpolates with unfused round-to-nearest ops and a float64
t = i/n exactly as the reference, and exits on ``__ballot_sync`` of an
invalid in-range lane.  The W-block count of the first failing state is
returned, so ``raked_motion_check``'s ``blocks`` equals the reference's for
the context's width.
"""

from __future__ import annotations

import math

import numpy as np

from . import runtime
from .collision import ValidationContext
from .lanes import Config


def _pair(start: Config, goal: Config) -> tuple[np.ndarray, np.ndarray]:
    s = np.asarray(start, dtype=np.float32).reshape(-1)
    g = np.asarray(goal, dtype=np.float32).reshape(-1)
    if s.shape != g.shape:
        raise ValueError(f"dimension mismatch: {s.shape[0]} vs {g.shape[0]}")
    return s, g


def _bind(ctx):
    """(robot module, device env) for any context exposing program/pairs/env
    (ours, or a reference ValidationContext built before patch_vecmp)."""
    mod = runtime.robot_module(ctx.program, ctx.pairs)
    return mod, runtime.device_env(ctx.env, mod.home)


def _check_resolution(resolution: float) -> None:
    if not resolution > 0:
        raise ValueError(f"resolution must be positive, got {resolution}")


def discretization_count(start: Config, goal: Config, resolution: float) -> int:
    """max(1, ceil(distance / resolution)) computed by the device kernel
    (reference motion.py:25-29)."""
    _check_resolution(resolution)
    s, g = _pair(start, goal)
    sd = runtime.to_device(s.reshape(1, -1))
    gd = runtime.to_device(g.reshape(1, -1))
    return int(runtime.discretize_device(sd, gd, resolution).cpu()[0])


def rake_strata(n: int, width: int) -> tuple[int, np.ndarray]:
    """Stratum length and base offsets (host integer helper, reference motion.py:32-35)."""
    s = math.ceil(n / width)
    return s, np.arange(width, dtype=np.int64) * s


def raked_motion_check(start: Config, goal: Config, ctx: ValidationContext,
                       resolution: float, backward: bool = False) -> tuple[bool, int]:
    """(verdict, block evaluations of a ctx.width-lane rake) - reference motion.py:38-78."""
    _check_resolution(resolution)
    s, g = _pair(start, goal)
    if s.shape[0] != ctx.program.dof:
        raise ValueError(f"block dim {s.shape[0]} != program dof {ctx.program.dof}")
    ctx.motion_checks += 1
    # one host-buffer C call: pinned staging -> begin + rake + finalize -> read-back
    verdict, _, blocks = runtime.motions_host(*_bind(ctx), s.reshape(1, -1), g.reshape(1, -1),
                                              resolution, width=ctx.width, backward=backward,
                                              prune=getattr(ctx, "prune", True))
    nblocks = int(blocks[0])
    ctx.blocks_evaluated += nblocks
    return bool(verdict[0]), nblocks


def validate_motion_rake(start: Config, goal: Config, ctx: ValidationContext,
                         resolution: float, backward: bool = False) -> bool:
    """True iff every state at i/n, i = 1..n, is valid (reference motion.py:81-90)."""
    verdict, _ = raked_motion_check(start, goal, ctx, resolution, backward)
    return verdict


class MotionValidator:
    """Fixed-size batched rake with device-resident buffers and a CUDA graph.

    For callers that validate many batches of ``n_edges`` edges (planner
    rounds, the benchmark): the begin, rake and finalize launches are captured once and
    replayed, so a call costs one graph launch.  ``__call__`` copies the edges
    into the resident buffers (from host memory - pinned for async copies - or
    from device tensors), replays, and returns the packed int32 verdict words
    on the device (``.host_bits()`` reads them back).
    """

    def __init__(self, ctx: ValidationContext, n_edges: int, resolution: float, *,
                 width: int = 32, backward: bool = False, graph: bool = True,
                 overlapped: bool = False):
        _check_resolution(resolution)
        torch = runtime.require_cuda()
        self.ctx, self.n_edges, self.resolution = ctx, int(n_edges), float(resolution)
        self.width, self.backward = int(width), bool(backward)
        self.overlapped = bool(overlapped)     # runs next to other batches (pipeline)
        dof = ctx.program.dof
        dev = torch.cuda.current_device()
        self.starts = torch.zeros((self.n_edges, dof), dtype=torch.float32, device=dev)
        self.goals = torch.zeros_like(self.starts)
        self.bits = torch.zeros(max((self.n_edges + 31) // 32, 1), dtype=torch.int32, device=dev)
        self.workspace = runtime.motion_workspace(self.n_edges)
        self._host_bits = torch.empty(self.bits.shape, dtype=torch.int32).pin_memory()
        self._mod, self._denv = _bind(ctx)
        self.graph = None
        if graph and self.n_edges:
            self._launch()                        # warm up (module load, occupancy query)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch()
            self.graph = g

    def _launch(self) -> None:
        runtime.validate_motions_device(self._mod, self._denv, self.starts, self.goals,
                                        self.resolution, width=self.width,
                                        backward=self.backward, prune=getattr(self.ctx, "prune", True),
                                        bits=self.bits, workspace=self.workspace,
                                        overlapped=self.overlapped)

    def __call__(self, starts=None, goals=None):
        if starts is not None:
            self.starts.copy_(runtime._as_tensor(starts), non_blocking=True)
            self.goals.copy_(runtime._as_tensor(goals), non_blocking=True)
        self.ctx.motion_checks += self.n_edges
        if self.graph is not None:
            self.graph.replay()
        elif self.n_edges:
            self._launch()
        return self.bits

    def host_bits(self):
        """Verdict words copied to pinned host memory (synchronises the stream)."""
        self._host_bits.copy_(self.bits, non_blocking=True)
        runtime.require_cuda().cuda.current_stream().synchronize()
        return self._host_bits.numpy()

    def verdicts(self) -> np.ndarray:
        return runtime.unpack_bits(self.host_bits(), self.n_edges)


_NO_STEP_GRAPH = __import__("os").environ.get("VMP_EXP_NO_STEP_GRAPH") is not None   # experiments


class MotionPipeline:
    """Multi-buffered stream of fixed-size edge batches from host memory.

    Each slot (a ``MotionValidator``: device buffers + CUDA graph) owns a
    stream, and ``submit(starts, goals)`` enqueues the whole step on it: the
    host->device copy of the batch, the graph replay (begin -> rake ->
    finalize) and the verdict read-back into the slot's pinned host buffer.
    Batches in different slots share no stream and no event, so batch k+1's
    copy and rake start while batch k's rake drains (measured: 41.6 us per
    4,096-edge config-2 step at depth 3 against 49.9 us for back-to-back
    replays on one stream, scripts/exp_pipe2.py).  ``result(ticket)`` waits
    for that batch and returns its verdict words in pinned host memory; a
    slot is reused after ``depth`` submits, which first waits for the slot's
    previous batch.  Every batch still pays its own H2D and D2H transfers -
    they are only overlapped with other batches' compute.  When the caller
    refills the same pinned host buffers every step, the whole step - both
    copies in, the three kernels, the copy out - is one CUDA graph per slot
    (keyed by the source pointers): one launch per step instead of five API
    calls (config 2: 35.3 -> 31.2 us per step end to end).
    """

    def __init__(self, ctx: ValidationContext, n_edges: int, resolution: float, *,
                 width: int = 32, depth: int = 3):
        torch = runtime.require_cuda()
        self.torch = torch
        self.slots = [MotionValidator(ctx, n_edges, resolution, width=width, overlapped=True)
                      for _ in range(depth)]
        self.streams = [torch.cuda.Stream() for _ in self.slots]
        origin = torch.cuda.current_stream()
        self.host = [torch.empty(s.bits.shape, dtype=torch.int32).pin_memory() for s in self.slots]
        self.done = [torch.cuda.Event() for _ in self.slots]
        for st, ev in zip(self.streams, self.done):
            st.wait_stream(origin)                              # buffers initialised
            ev.record(st)
        self.count = 0
        # whole-step graphs (H2D copies + begin / rake / finalize + D2H copy) per
        # slot, keyed by the pinned source buffers: a caller that refills the same
        # pinned buffers every step pays one graph launch per step
        self._step_graphs = [dict() for _ in self.slots]

    def _step_graph(self, k: int, hs, hg):
        """The slot's whole-step graph for these pinned source tensors, or None."""
        if not (hs.is_pinned() and hg.is_pinned()) or self.slots[k].graph is None or _NO_STEP_GRAPH:
            return None
        key = (hs.data_ptr(), hg.data_ptr(), tuple(hs.shape), tuple(hg.shape))
        cache = self._step_graphs[k]
        if key not in cache:
            if len(cache) >= 4:                                 # callers with ever-new buffers
                return None
            slot, st = self.slots[k], self.streams[k]
            g = self.torch.cuda.CUDAGraph()
            with self.torch.cuda.graph(g, stream=st):
                slot.starts.copy_(hs, non_blocking=True)
                slot.goals.copy_(hg, non_blocking=True)
                slot._launch()
                self.host[k].copy_(slot.bits, non_blocking=True)
            cache[key] = (g, hs, hg)                            # keeps the buffers alive
        return cache[key][0]

    def submit(self, starts, goals) -> int:
        k = self.count % len(self.slots)
        slot, st = self.slots[k], self.streams[k]
        if self.count >= len(self.slots):
            self.done[k].synchronize()                          # slot's previous batch is out
        hs, hg = runtime._as_tensor(starts), runtime._as_tensor(goals)
        whole = self._step_graph(k, hs, hg) if not hs.is_cuda and not hg.is_cuda else None
        with self.torch.cuda.stream(st):
            if whole is not None:
                slot.ctx.motion_checks += slot.n_edges
                whole.replay()                                  # copies + kernels: one launch
            else:
                slot.starts.copy_(hs, non_blocking=True)
                slot.goals.copy_(hg, non_blocking=True)
                slot()                                          # graph replay on the slot's stream
                self.host[k].copy_(slot.bits, non_blocking=True)
            self.done[k].record(st)
        self.count += 1
        return self.count - 1

    def wait_all(self, stream=None) -> None:
        """Make ``stream`` (default: the current one) wait for every submitted batch."""
        stream = stream or self.torch.cuda.current_stream()
        for st in self.streams:
            stream.wait_stream(st)

    def result(self, ticket: int):
        """Verdict words of batch ``ticket``; only the last ``depth`` batches are held
        (a slot's buffer is overwritten by the submit ``depth`` tickets later)."""
        if not (self.count - len(self.slots) <= ticket < self.count):
            raise ValueError(f"ticket {ticket} is not held: the pipeline holds the last "
                             f"{len(self.slots)} batches ({max(self.count - len(self.slots), 0)}"
                             f"..{self.count - 1})")
        k = ticket % len(self.slots)
        self.done[k].synchronize()
        return self.host[k].numpy()


def validate_motions(ctx: ValidationContext, starts, goals, resolution: float, *,
                     backward: bool = False, width: int = 32, counts: bool = False,
                     bits=None, workspace=None):
    """Batched rake over E edges in one launch (new entry point).

    ``starts``/``goals``: (E, dof) float32 (numpy or CUDA tensors).  Returns
    packed int32 verdict words on the device, plus per-edge
    (n_states, blocks) device tensors when ``counts``.
    """
    _check_resolution(resolution)
    sd = runtime.to_device(starts)
    gd = runtime.to_device(goals)
    if sd.shape != gd.shape:
        raise ValueError(f"starts {tuple(sd.shape)} and goals {tuple(gd.shape)} differ")
    if sd.dim() != 2 or sd.shape[1] != ctx.program.dof:
        raise ValueError(f"edges must be (E, dof={ctx.program.dof}), got {tuple(sd.shape)}")
    sd = sd.contiguous()
    gd = gd.contiguous()
    ctx.motion_checks += sd.shape[0]
    b, n_states, blocks = runtime.validate_motions_device(
        *_bind(ctx), sd, gd, resolution, width=width, backward=backward,
        prune=getattr(ctx, "prune", True), want_counts=counts, bits=bits, workspace=workspace)
    return (b, n_states, blocks) if counts else b
