"""pytest plugin: run the REFERENCE's own test-suite with the hot path on the GPU.

Loaded with `-p vmp_patch_plugin` before the reference conftest imports its
names, so every ValidationContext / validate_block / evaluate_program /
motion call in the reference's tests, planners and CLI goes through
paper_2309_14545_b200 (see paper_2309_14545_b200/install.py).  The terminal
summary lists how many calls each replacement served."""
import vecmp

from paper_2309_14545_b200 import install

PATCHED = install.patch_vecmp(vecmp, count=True)


def pytest_report_header(config):
    return f"vmp: patched {len(PATCHED)} reference names onto the B200 path"


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"vmp: patched {len(PATCHED)} names: {', '.join(PATCHED)}")
    calls = ", ".join(f"{k}={v}" for k, v in sorted(install.CALLS.items()))
    terminalreporter.write_line(f"vmp: calls served by the B200 path: {calls}")
