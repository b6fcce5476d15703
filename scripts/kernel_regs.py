"""Registers / local memory of the NVRTC-compiled robot kernels (no GPU needed).

    python scripts/kernel_regs.py [repo]
"""
import sys, subprocess, re, tempfile, os
sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else "/root/repo")
from paper_2309_14545_b200 import load_robot, codegen
from paper_2309_14545_b200._native import lib, check
for name in ("arm7", "fetch_standin", "baxter_standin"):
    r = load_robot(name)
    src = codegen.generate_source(r.program, r.pairs, name)
    out = f"/tmp/{name}_nvrtc.cubin"
    check(lib().vmp_compile(src.encode(), f"{name}.cu".encode(), out.encode()))
    ru = subprocess.run(["cuobjdump", "--dump-resource-usage", out], capture_output=True, text=True).stdout
    for m in re.finditer(r"Function (vmp_motion_p1_s2_g1\w*|vmp_validate_p1_s1_g1)\b.*?\n.*?REG:(\d+) STACK:(\d+)", ru):
        print(name, m.group(1), "REG", m.group(2), "STACK", m.group(3))
