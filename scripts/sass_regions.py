"""Split an ncu source-page CSV (--page source --csv --print-source sass) into runs
of instructions with the same execution count: executed warp instructions, share
of the kernel and opcode mix per run (where does the instruction budget go?).

    python scripts/sass_regions.py page.csv [min_share_pct]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
min_share = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
i_e, i_s = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ex = [float(r[i_e] or 0) for r in data]
st = [float(r[i_s] or 0) for r in data]
tot, tot_s = sum(ex), sum(st)


def opcode(src):
    t = src.split()
    op = t[1] if t[0].startswith("@") else t[0]
    return op.split(".")[0]


runs, start = [], 0
for k in range(1, len(data) + 1):
    if k == len(data) or abs(ex[k] - ex[start]) > 0.02 * max(ex[start], 1):
        runs.append((start, k))
        start = k
print(f"total warp instructions {tot:,.0f}; samples {tot_s:,.0f}")
for a, b in runs:
    e = sum(ex[a:b])
    if e / tot * 100 < min_share:
        continue
    mix = Counter(opcode(data[k][1]) for k in range(a, b))
    top = " ".join(f"{o}:{c}" for o, c in mix.most_common(7))
    print(f"[{a:5d},{b:5d}) n={b - a:4d} exec/instr={ex[a]:>11,.0f} share={e / tot * 100:5.1f}% "
          f"stall-share={sum(st[a:b]) / tot_s * 100:5.1f}%  {top}")
