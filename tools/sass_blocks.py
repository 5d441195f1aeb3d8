"""Hot SASS of one kernel in an .ncu-rep source page: opcode mix and the
basic blocks (runs of equal execution count) above 1% of the instructions.
    python tools/sass_blocks.py report.ncu-rep [kernel-substring] [--dump]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
secs = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
secs.append(len(rows))
for a, b in zip(secs, secs[1:]):
    name = rows[a][1]
    if sub not in name:
        continue
    hdr = rows[a + 1]
    ie, si = hdr.index("Instructions Executed"), hdr.index("Source")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[a + 2:b] if len(r) > ie and r[ie].isdigit()]
    tot = sum(int(r[ie]) for r in data)
    print(f"== {name[:100]}\n   {tot} warp instructions")
    op = collections.Counter()
    for r in data:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[si])
        op[m.group(2) if m else "?"] += int(r[ie])
    print("  ", ", ".join(f"{o}={c / tot * 100:.1f}%" for o, c in op.most_common(20)))
    cur, n, start, stall = None, 0, None, 0
    for r in data + [["", "", "0", "", "", "-1"] + [""] * 10]:
        c = int(r[ie]) if r[ie].lstrip("-").isdigit() else -1
        if c != cur:
            if cur is not None and cur * n > tot * 0.01:
                print(f"   {start} n={n:4d} x{cur:9d} {cur * n / tot * 100:5.1f}%  stall={stall}")
            cur, n, start, stall = c, 0, r[0][-5:], 0
        n += 1
        stall += int(r[st]) if r[st].isdigit() else 0
    if "--dump" in sys.argv:
        for r in data:
            if int(r[ie]) > 0:
                print(f"{r[0][-5:]} {int(r[ie]):9d} {r[st]:>5s} {r[si][:90]}")
