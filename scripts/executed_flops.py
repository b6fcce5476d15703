"""Executed FP32 flop per launch from an ncu capture's SASS source page.

ncu's op counters (smsp__sass_thread_inst_executed_op_ffma_pred_on ...) do not
count the packed FFMA2 / FADD2 / FMUL2 of sm_100, so this sums the
predicated-on thread instructions of every SASS line by opcode: FFMA 2 flop,
FADD / FMUL 1, FFMA2 4, FADD2 / FMUL2 2 (MUFU, FMNMX, FSETP are not counted).

    python scripts/executed_flops.py gpurun_out/prof_motion.ncu-rep [...]
"""
import csv
import io
import json
import re
import subprocess
import sys

FLOPS = {"FFMA": 2, "FADD": 1, "FMUL": 1, "FFMA2": 4, "FADD2": 2, "FMUL2": 2}


def executed(path: str) -> dict:
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_src = hdr.index("Source")
    i_on = hdr.index("Predicated-On Thread Instructions Executed")
    flop = 0
    by = {}
    for r in rows[2:]:
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9]+)(?:\.[A-Z0-9_.]+)?\s", r[i_src] + " ")
        if not m:
            continue
        op = m.group(1)
        if op in FLOPS:
            n = float(r[i_on] or 0)
            by[op] = by.get(op, 0) + n
            flop += FLOPS[op] * n
    return {"flop_per_launch": flop, "thread_inst": by}


if __name__ == "__main__":
    print(json.dumps({p: executed(p) for p in sys.argv[1:]}, indent=1))
