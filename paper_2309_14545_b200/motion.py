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
    return (runtime.robot_module(ctx.program, ctx.pairs), runtime.device_env(ctx.env))


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
    sd = runtime.to_device(s.reshape(1, -1))
    gd = runtime.to_device(g.reshape(1, -1))
    bits, _, blocks = runtime.validate_motions_device(
        *_bind(ctx), sd, gd, resolution, width=ctx.width, backward=backward,
        prune=getattr(ctx, "prune", True), want_counts=True)
    verdict = bool(int(bits[0].item()) & 1)
    nblocks = int(blocks[0].item())
    ctx.blocks_evaluated += nblocks
    return verdict, nblocks


def validate_motion_rake(start: Config, goal: Config, ctx: ValidationContext,
                         resolution: float, backward: bool = False) -> bool:
    """True iff every state at i/n, i = 1..n, is valid (reference motion.py:81-90)."""
    verdict, _ = raked_motion_check(start, goal, ctx, resolution, backward)
    return verdict


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
