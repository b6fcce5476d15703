"""Summarise .ncu-rep captures into markdown (run in the build container).

    python scripts/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/roundN_ncu.md
"""

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %", 1),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %", 1),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
    ("launch__registers_per_thread", "registers", 1),
    ("launch__grid_size", "grid", 1),
    ("smsp__inst_executed.sum", "warp instructions", 1),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / instr", 1),
    ("dram__bytes_read.sum", "DRAM read", 1),
    ("dram__bytes_write.sum", "DRAM write", 1),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected", 1),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait", 1),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb", 1),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_sb", 1),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "stall no_instr", 1),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall dispatch", 1),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def fmt(v, unit, scale):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    text = f"{x:,.2f}" if abs(x) < 1e6 else f"{x:,.0f}"
    return f"{text} {unit}".strip() if unit and unit not in ("%", "register/thread") else text


def main(paths):
    print("| metric | " + " | ".join(p.split("/")[-1].replace(".ncu-rep", "") for p in paths) + " |")
    print("|---|" + "---|" * len(paths))
    data = [raw(p)[0] for p in paths]
    print("| kernel | " + " | ".join(d[0].get("Kernel Name", "?")[:40] for d in data) + " |")
    for key, label, scale in METRICS:
        cells = [fmt(d[0].get(key, "-"), d[1].get(key, ""), scale) for d in data]
        print(f"| {label} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
