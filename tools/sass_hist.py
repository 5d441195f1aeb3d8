"""Opcode histogram (executed warp instructions, stall samples) and the
hottest SASS lines of one kernel in an .ncu-rep (source page):
    python tools/sass_hist.py report.ncu-rep [min_count]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ei, si, st = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
pi = hdr.index("Avg. Predicated-On Threads Executed")
data = rows[2:]
tot = sum(int(r[ei] or 0) for r in data)
stot = sum(int(r[st] or 0) for r in data)
op, stall = collections.Counter(), collections.Counter()
for r in data:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[si])
    o = m.group(2) if m else "?"
    op[o] += int(r[ei] or 0)
    stall[o] += int(r[st] or 0)
print(f"total {tot} warp instructions, {stot} stall samples")
for o, c in op.most_common(25):
    print(f"{o:10s} {c / tot * 100:5.1f}%  stall {stall[o] / max(stot, 1) * 100:5.1f}%")
if mn:
    for i, r in enumerate(data):
        if int(r[ei] or 0) >= mn or int(r[st] or 0) >= stot / 100:
            print(i, r[ei], r[pi], r[st], r[si][:80])
