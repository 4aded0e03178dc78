"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA line.

usage: ncu -i REP --page source --csv --print-source cuda,sass -k regex:K -c 1 > x.csv
       python scripts/ncu_lines.py x.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file = None
hdr = None
lines = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samples = int(r[4])
        execd = int(r[7])
        thr = float(r[10])
    except (ValueError, IndexError):
        continue
    lines.append((samples, execd, thr, cur_file, r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in lines) or 1
tex = sum(x[1] for x in lines) or 1
print(f"total samples {tot}, executed warp-instructions {tex}")
for s, e, t, f, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% smp {100*e/tex:5.1f}% ex thr{t:5.1f} {f}:{ln:5s} {src}")
