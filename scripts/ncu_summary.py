"""Key ncu metrics per launch from a .ncu-rep (raw page), one line per kernel.

usage: python scripts/ncu_summary.py REPORT.ncu-rep [more metric names...]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
extra = sys.argv[2:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum"] + extra
short = ["us", "rdMB", "wrMB", "regs", "occ%", "issue%", "L2hit", "L1hit", "fp64%", "inst"] + extra
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:60]
    vals = []
    for w, s in zip(want, short):
        if w in h:
            vals.append(f"{s}={r[h.index(w)]}")
    print(name, " ".join(vals))
