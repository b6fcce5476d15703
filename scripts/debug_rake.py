import sys
from pathlib import Path
sys.path[:0] = [str(Path(__file__).resolve().parents[1]), str(Path(__file__).resolve().parents[1] / "tests")]
import numpy as np, torch
import golden_io
from paper_2309_14545_b200 import ValidationContext, load_robot, runtime
from paper_2309_14545_b200 import motion as M
fx = golden_io.load("motion"); key = "arm7_0"
rob = load_robot("arm7"); env = golden_io.env_from(fx, f"env_{key}")
s, g, res = fx[f"starts_{key}"], fx[f"goals_{key}"], float(fx[f"res_{key}"])
ctx = ValidationContext(rob.program, rob.model, rob.pairs, env, width=8)
bad = 0
for i in range(len(s)):
    got = M.raked_motion_check(s[i], g[i], ctx, res)
    exp = (bool(fx[f"verdict_{key}_w8_b0"][i]), int(fx[f"blocks_{key}_w8_b0"][i]))
    if got != exp:
        bad += 1
        if bad < 6: print("edge", i, "got", got, "exp", exp, "n", int(fx[f"n_{key}"][i]))
print("per-edge mismatches", bad, "of", len(s))
# same edge set, batched with a reused workspace, twice
ws = runtime.motion_workspace(len(s))
for rep in range(3):
    b, n, blk = M.validate_motions(ctx, s, g, res, width=8, counts=True, workspace=ws)
    v = runtime.unpack_bits(b.cpu().numpy(), len(s))
    print("batched rep", rep, "verdict mism", int((v != fx[f"verdict_{key}_w8_b0"]).sum()),
          "blocks mism", int((blk.cpu().numpy() != fx[f"blocks_{key}_w8_b0"]).sum()))
# single edge repeated with reused workspace
ws1 = runtime.motion_workspace(1)
for i in range(0, 40, 9):
    b, n, blk = M.validate_motions(ctx, s[i:i+1], g[i:i+1], res, width=8, counts=True, workspace=ws1)
    print("single", i, int(b[0].item()) & 1, int(blk[0].item()), "exp", fx[f"verdict_{key}_w8_b0"][i], fx[f"blocks_{key}_w8_b0"][i])
# the exact sequence of tests/test_gpu_parity.py::test_rake_vs_reference_goldens
for rep in range(5):
    bad = 0
    for width in (8, 1, 32):
        for bwd in (0, 1):
            c2 = ValidationContext(rob.program, rob.model, rob.pairs, env, width=width)
            b, n, blk = M.validate_motions(c2, s, g, res, backward=bool(bwd), width=width, counts=True)
            v = runtime.unpack_bits(b.cpu().numpy(), len(s))
            bad += int((v != fx[f"verdict_{key}_w{width}_b{bwd}"]).sum())
    c8 = ValidationContext(rob.program, rob.model, rob.pairs, env, width=8)
    for i in range(0, len(s), 9):
        if M.raked_motion_check(s[i], g[i], c8, res) != (bool(fx[f"verdict_{key}_w8_b0"][i]), int(fx[f"blocks_{key}_w8_b0"][i])):
            bad += 1
            print("  rep", rep, "edge", i, "MISMATCH")
    print("sequence rep", rep, "mismatches", bad)
