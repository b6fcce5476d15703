import sys, os
from pathlib import Path
sys.path[:0] = [str(Path(__file__).resolve().parents[1]), str(Path(__file__).resolve().parents[1] / "tests")]
import numpy as np, torch
import golden_io
from paper_2309_14545_b200 import ValidationContext, load_robot, runtime
from paper_2309_14545_b200 import motion as M
fx = golden_io.load("motion"); key = "arm7_0"
rob = load_robot("arm7"); env = golden_io.env_from(fx, f"env_{key}")
s, g, res = fx[f"starts_{key}"], fx[f"goals_{key}"], float(fx[f"res_{key}"])
tag = os.environ.get("TAG", "")
for rep in range(4):
    out = []
    for width in (8, 1, 32):
        for bwd in (0, 1):
            c2 = ValidationContext(rob.program, rob.model, rob.pairs, env, width=width)
            b, n, blk = M.validate_motions(c2, s, g, res, backward=bool(bwd), width=width, counts=True)
            v = runtime.unpack_bits(b.cpu().numpy(), len(s))
            nb = int((v != fx[f"verdict_{key}_w{width}_b{bwd}"]).sum())
            nn = int((n.cpu().numpy() != fx[f"n_{key}"]).sum())
            out.append(f"w{width}b{bwd}:{nb}/{nn}")
    print(tag, "rep", rep, " ".join(out), flush=True)
