"""Opcode histogram of one kernel's SASS (cuobjdump), for instruction-count
work before spending GPU time.

usage: python scripts/sass_hist.py LIB.so NAME_SUBSTRING [top]
"""
import re
import subprocess
import sys
from collections import Counter

lib, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = Counter()
    for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[T0-9]\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", f):
        ops[m.group(1)] += 1
    total = sum(ops.values())
    fp64 = sum(v for k, v in ops.items() if k.startswith("D") and k not in ("DEPBAR",))
    print(f"{name[:110]}\n  total {total}  fp64 {fp64}  " +
          " ".join(f"{k}:{v}" for k, v in ops.most_common(top)))
