"""Aggregate an ncu source page (SASS view, --page source --csv) of one
kernel: executed warp instructions and stall samples per opcode, and the
hottest instructions.

usage: ncu -i REP --page source --csv -k regex:NAME > x.csv
       python scripts/ncu_sass_hot.py x.csv [top]
"""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
h = rows[1]
ia, isrc = h.index("Address"), h.index("Source")
iex = h.index("Instructions Executed")
ist = h.index("Warp Stall Sampling (All Samples)")
ops, stalls = Counter(), Counter()
lines = []
for r in rows[2:]:
    if len(r) < len(h) or r[iex] == "Instructions Executed":
        continue
    src = r[isrc].strip()
    tok = src.split()
    if not tok:
        continue
    op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
    op = op.split(".")[0]
    ex = int(float(r[iex] or 0))
    st = int(float(r[ist] or 0))
    ops[op] += ex
    stalls[op] += st
    lines.append((st, ex, r[ia][-5:], src[:90]))
tot = sum(ops.values())
print("executed warp instructions", tot, " stall samples", sum(stalls.values()))
for op, n in ops.most_common(top):
    print(f"  {op:10s} {n:10d} {100.0 * n / tot:5.1f}%  stalls {stalls[op]}")
print("hottest instructions (stall samples):")
for st, ex, a, s in sorted(lines, reverse=True)[:top]:
    print(f"  {st:6d} {ex:9d} {a} {s}")
