"""Drop the B200 path into an imported reference package (``vecmp``).

    import vecmp
    from paper_2309_14545_b200.install import patch_vecmp
    patch_vecmp(vecmp)

Rebinds the hot-path names everywhere the reference binds them - its own
modules import them by value at import time (planners.py:18,21,
simplify.py:17,19, cli.py:22,24) - so the reference's
planners, simplifier, CLI/RPC and tests run their FK, collision checks and
motion validation on the GPU; ``shortcut`` / ``bspline_smooth`` /
``simplify_path``, ``prm`` and ``rrt_connect`` are replaced by their batched
versions (simplify.py, prm.py, rrt.py - identical results, checked against
reference runs).
Host-side types (ConfigBlock, Environment,
primitives, KinematicProgram) stay the reference's own; the shims duck-type
them.  ``unpatch`` restores the originals.
"""

from __future__ import annotations

import importlib

from . import collision, motion, program, simplify

#: module -> names to rebind (only where the module actually defines them)
TARGETS = {
    "": ("evaluate_program", "validate_block", "ValidationContext", "sphere_vs_sphere_lanes",
         "sphere_vs_capsule_lanes", "sphere_vs_cuboid_lanes", "discretization_count",
         "raked_motion_check", "validate_motion_rake", "shortcut", "bspline_smooth",
         "simplify_path"),
    "program": ("evaluate_program",),
    "collision": ("evaluate_program", "validate_block", "ValidationContext",
                  "sphere_vs_sphere_lanes", "sphere_vs_capsule_lanes", "sphere_vs_cuboid_lanes"),
    "motion": ("ValidationContext", "discretization_count", "raked_motion_check",
               "validate_motion_rake"),
    "planners": ("ValidationContext", "validate_motion_rake"),
    "simplify": ("ValidationContext", "validate_motion_rake", "shortcut", "bspline_smooth",
                 "simplify_path"),
    "cli": ("ValidationContext", "validate_motion_rake", "simplify_path"),
    "bench": ("simplify_path",),
}

REPLACEMENTS = {
    "evaluate_program": program.evaluate_program,
    "validate_block": collision.validate_block,
    "ValidationContext": collision.ValidationContext,
    "sphere_vs_sphere_lanes": collision.sphere_vs_sphere_lanes,
    "sphere_vs_capsule_lanes": collision.sphere_vs_capsule_lanes,
    "sphere_vs_cuboid_lanes": collision.sphere_vs_cuboid_lanes,
    "discretization_count": motion.discretization_count,
    "raked_motion_check": motion.raked_motion_check,
    "validate_motion_rake": motion.validate_motion_rake,
    # batched speculative simplifier: same waypoints, motion checks in launches
    "shortcut": simplify.shortcut,
    "bspline_smooth": simplify.bspline_smooth,
    "simplify_path": simplify.simplify_path,
}

#: names whose replacement is built against the patched package's own types
ADAPTED = {"": ("prm", "rrt_connect"), "planners": ("prm", "rrt_connect"),
           "bench": ("prm", "rrt_connect")}


def reference_prm(pkg):
    """A drop-in for the reference ``prm(problem, settings)`` (planners.py:243-291)
    running round-batched on the device (prm.prm_rounds): same waypoints,
    iterations and ValidationContext counters, the reference's own Path /
    PlanResult / InvalidProblemError types."""
    planners = importlib.import_module(f"{pkg.__name__}.planners")
    from . import prm as batched

    def prm(problem, settings=None):
        settings = settings or planners.PlannerSettings()
        st = batched.PRMSettings(resolution=settings.resolution,
                                 max_iterations=settings.max_iterations, prm_k=settings.prm_k,
                                 prm_batch=settings.prm_batch,
                                 rake_backward=settings.rake_backward, width=settings.width)
        try:
            res = batched.prm_rounds(problem.robot, problem.env, problem.start, problem.goal, st)
        except batched.InvalidProblemError as exc:
            raise planners.InvalidProblemError(str(exc)) from None
        path = planners.Path(list(res.waypoints)) if res.success else None
        return planners.PlanResult(path, iterations=res.iterations,
                                   blocks_evaluated=res.blocks_evaluated,
                                   motion_checks=res.motion_checks)
    prm.__doc__ = reference_prm.__doc__
    return prm


def reference_rrt_connect(pkg):
    """A drop-in for the reference ``rrt_connect(problem, settings)``
    (planners.py:180-210) with batched connect chains (rrt.rrt_connect_batched):
    same waypoints, iterations and counters, the reference's own types."""
    planners = importlib.import_module(f"{pkg.__name__}.planners")
    from . import prm as batched_prm
    from . import rrt as batched

    def rrt_connect(problem, settings=None):
        settings = settings or planners.PlannerSettings()
        st = batched.RRTSettings(resolution=settings.resolution, range=settings.range,
                                 max_iterations=settings.max_iterations,
                                 rake_backward=settings.rake_backward, width=settings.width)
        try:
            res = batched.rrt_connect_batched(problem.robot, problem.env, problem.start,
                                              problem.goal, st)
        except batched_prm.InvalidProblemError as exc:
            raise planners.InvalidProblemError(str(exc)) from None
        path = planners.Path(list(res.waypoints)) if res.success else None
        return planners.PlanResult(path, iterations=res.iterations,
                                   blocks_evaluated=res.blocks_evaluated,
                                   motion_checks=res.motion_checks)
    rrt_connect.__doc__ = reference_rrt_connect.__doc__
    return rrt_connect


_SAVED: dict = {}
#: calls routed to the B200 path per name (filled when patched with count=True)
CALLS: dict = {}


def _counting(name, fn):
    if isinstance(fn, type):
        class Counted(fn):
            def __init__(self, *args, **kwargs):
                CALLS[name] = CALLS.get(name, 0) + 1
                super().__init__(*args, **kwargs)
        Counted.__name__ = Counted.__qualname__ = fn.__name__
        return Counted

    def wrapper(*args, **kwargs):
        CALLS[name] = CALLS.get(name, 0) + 1
        return fn(*args, **kwargs)
    wrapper.__name__ = fn.__name__
    wrapper.__doc__ = fn.__doc__
    return wrapper


def patch_vecmp(pkg, count: bool = False) -> list[str]:
    """Rebind the hot-path names in ``pkg`` (the imported vecmp package).

    With ``count`` every replacement is wrapped to tally its calls in CALLS.
    """
    done = []
    table = {k: (_counting(k, v) if count else v) for k, v in REPLACEMENTS.items()}
    for name, make in (("prm", reference_prm), ("rrt_connect", reference_rrt_connect)):
        adapted = make(pkg)
        table[name] = _counting(name, adapted) if count else adapted
    targets = {sub: TARGETS.get(sub, ()) + ADAPTED.get(sub, ()) for sub in {**TARGETS, **ADAPTED}}
    for sub, names in targets.items():
        try:
            mod = importlib.import_module(f"{pkg.__name__}.{sub}") if sub else pkg
        except ImportError:
            continue
        for name in names:
            if hasattr(mod, name):
                _SAVED.setdefault((mod.__name__, name), getattr(mod, name))
                setattr(mod, name, table[name])
                done.append(f"{mod.__name__}.{name}")
    return done


def unpatch_vecmp(pkg) -> None:
    for (modname, name), original in list(_SAVED.items()):
        mod = importlib.import_module(modname)
        setattr(mod, name, original)
    _SAVED.clear()
