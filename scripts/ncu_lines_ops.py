"""Per source line of one kernel: executed warp instructions, and how many of
them are register moves (IMAD.MOV / MOV), fp64 selects (FSEL) and fp64 math,
from an ncu source page exported with --print-source sass,cuda.

usage: ncu -i REP --page source --csv --print-source sass,cuda --launch-skip K --launch-count 1 > x.csv
       python scripts/ncu_lines_ops.py x.csv [top]
"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
cur_file, cur_line, cur_src = "?", "?", ""
agg = defaultdict(lambda: defaultdict(int))
src_text = {}
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":  # a source line
        cur_line, cur_src = r[0], r[1]
        src_text[(cur_file, cur_line)] = cur_src.strip()[:90]
        continue
    sass = r[3]
    try:
        n = int(r[7])
    except ValueError:
        continue
    m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", sass)
    op = m.group(1) if m else "?"
    a = agg[(cur_file, cur_line)]
    a["all"] += n
    if op.startswith("IMAD.MOV") or op == "MOV":
        a["mov"] += n
    if op == "FSEL" or op == "SEL":
        a["sel"] += n
    if op.startswith(("DADD", "DMUL", "DFMA")):
        a["fp64"] += n
tot = sum(a["all"] for a in agg.values())
print(f"total warp instr {tot}; moves {sum(a['mov'] for a in agg.values())}; selects {sum(a['sel'] for a in agg.values())}")
for (f, l), a in sorted(agg.items(), key=lambda kv: -kv[1]["all"])[:top]:
    print(f"{a['all']:10d} {100 * a['all'] / tot:5.1f}%  mov {a['mov']:9d} sel {a['sel']:9d} fp64 {a['fp64']:9d}  {f}:{l}  {src_text.get((f, l), '')}")
