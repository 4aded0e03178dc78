"""Per-source-line instruction counts and stall samples of one kernel:
joins ncu's per-SASS-instruction source page (executed instructions, stall
samples; in program order) with nvdisasm's line table of the same binary
(-g -c: "//## File ..., line N" annotations, innermost inlined line).

usage: python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX CUBIN MANGLED_SUBSTRING [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre, cubin, fsub = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
iex, ist, isrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
prof = []
for r in rows[2:]:
    if len(r) < len(h) or r[iex] == "Instructions Executed":
        if prof:
            break  # first launch only
        continue
    prof.append((int(float(r[iex] or 0)), int(float(r[ist] or 0)), r[isrc].strip()))
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = None
lines = []
cur = "?"
for ln in dis.splitlines():
    if ln.startswith("//-----") and ".text." in ln:
        sec = ln
        continue
    if sec is None or fsub not in sec:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m2 = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[T0-9]\s+)?([A-Z][A-Z0-9_]*)", ln)
    if m2 and not ln.strip().startswith("//"):
        lines.append((cur, m2.group(1)))


def opc(sass):
    t = sass.split()
    if not t:
        return ""
    o = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    return o.split(".")[0]


import difflib  # noqa: E402
a = [opc(p[2]) for p in prof]
b = [x[1] for x in lines]
sm = difflib.SequenceMatcher(a=a, b=b, autojunk=False)
agg = collections.Counter()
stall = collections.Counter()
matched = 0
for blk in sm.get_matching_blocks():
    for k in range(blk.size):
        key = lines[blk.b + k][0]
        agg[key] += prof[blk.a + k][0]
        stall[key] += prof[blk.a + k][1]
        matched += 1
print(f"sass rows: ncu {len(prof)}, nvdisasm {len(lines)}, aligned {matched}")
tot = sum(agg.values())
ts = sum(stall.values()) or 1
for key, v in agg.most_common(top):
    print(f"{100.0 * v / tot:5.1f}% instr  {100.0 * stall[key] / ts:5.1f}% stalls  {key}")
