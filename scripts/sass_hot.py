"""Hot SASS instructions of an ncu source-page CSV (--page source --csv
--print-source sass) with their dominant stall reasons.

    python scripts/sass_hot.py page.csv [lo hi]    (instruction index window)
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else len(data)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
stalls = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[i_s] or 0) for r in data)
for k in range(lo, hi):
    r = data[k]
    s = float(r[i_s] or 0)
    if s / tot < 0.002:
        continue
    top = sorted(((float(r[i] or 0), h[6:]) for i, h in stalls), reverse=True)[:3]
    print(f"{k:5d} {s / tot * 100:5.2f}% ex={r[i_e]:>8} {r[1][:60]:60s} "
          + " ".join(f"{h}:{v:.0f}" for v, h in top if v))
