"""patch_vecmp rebinds every import site of the reference (no GPU calls).

Uses the reference package from /root/reference when present (the build
container); skipped elsewhere - the GPU box runs the reference's whole suite
through scripts/run_reference_suite.sh instead."""

import importlib
import sys
from pathlib import Path

import pytest

REF_SRC = Path("/root/reference/pkg/src")


@pytest.fixture()
def vecmp_pkg():
    if not REF_SRC.exists():
        pytest.skip("reference package not available")
    sys.path.insert(0, str(REF_SRC))
    try:
        import vecmp
        yield vecmp
    finally:
        from paper_2309_14545_b200 import install
        install.unpatch_vecmp(vecmp)
        sys.path.remove(str(REF_SRC))


def test_patch_rebinds_all_import_sites(vecmp_pkg):
    from paper_2309_14545_b200 import collision, install, motion, program
    from paper_2309_14545_b200 import simplify as batched
    done = install.patch_vecmp(vecmp_pkg)
    assert len(done) == 40
    planners = importlib.import_module("vecmp.planners")
    simplify = importlib.import_module("vecmp.simplify")
    cli = importlib.import_module("vecmp.cli")
    assert planners.ValidationContext is collision.ValidationContext
    assert planners.validate_motion_rake is motion.validate_motion_rake
    assert simplify.validate_motion_rake is motion.validate_motion_rake
    assert cli.ValidationContext is collision.ValidationContext
    assert cli.simplify_path is batched.simplify_path
    assert importlib.import_module("vecmp.bench").simplify_path is batched.simplify_path
    assert vecmp_pkg.shortcut is batched.shortcut and simplify.bspline_smooth is batched.bspline_smooth
    assert vecmp_pkg.prm is planners.prm and "round-batched" in planners.prm.__doc__
    assert vecmp_pkg.rrt_connect is planners.rrt_connect
    assert "batched connect" in planners.rrt_connect.__doc__
    assert vecmp_pkg.program.evaluate_program is program.evaluate_program
    assert vecmp_pkg.collision.validate_block is collision.validate_block
    install.unpatch_vecmp(vecmp_pkg)
    assert planners.ValidationContext is not collision.ValidationContext


def test_counting_patch_keeps_signatures(vecmp_pkg):
    from paper_2309_14545_b200 import install
    install.patch_vecmp(vecmp_pkg, count=True)
    ctx_cls = vecmp_pkg.collision.ValidationContext
    assert issubclass(ctx_cls, install.REPLACEMENTS["ValidationContext"])
