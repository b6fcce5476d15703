"""pytest plugin: run the REFERENCE's own test-suite with the hot path on the GPU.

Loaded with `-p vmp_patch_plugin` before the reference conftest imports its
names, so every ValidationContext / validate_block / evaluate_program /
motion call in the reference's tests, planners and CLI goes through
paper_2309_14545_b200 (see paper_2309_14545_b200/install.py)."""
import vecmp

from paper_2309_14545_b200.install import patch_vecmp

PATCHED = patch_vecmp(vecmp)


def pytest_report_header(config):
    return f"vmp: patched {len(PATCHED)} reference names onto the B200 path"
