"""Aggregate an ncu report's SASS instruction counts (or, with --stalls, warp
stall samples) by CUDA source line:
    python tools/ncu_lines.py report.ncu-rep kernel_regex [top] [--stalls]"""
import collections
import csv
import io
import subprocess
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
rep, kern = args[0], args[1]
top = int(args[2]) if len(args) > 2 else 30
col = "Warp Stall Sampling (All Samples)" if "--stalls" in sys.argv else "Instructions Executed"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if col in r)
ei = hdr.index(col)
agg = collections.Counter()
text = {}
cur = None
fname = "?"
for r in rows:
    if r and r[0] == "File Path" and len(r) > 1:
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) <= ei or r is hdr:
        continue
    if r[0]:
        cur = (fname, int(r[0])) if r[0].isdigit() else cur
        text[cur] = r[1]
    try:
        n = int(r[ei])
    except ValueError:
        continue
    if r[2]:  # a SASS row (has an address)
        agg[cur] += n
tot = sum(agg.values())
print("total", tot)
for ln, n in agg.most_common(top):
    where = f"{ln[0]}:{ln[1]}" if ln else "?"
    print(f"{100 * n / tot:5.1f}% {n:>12d}  {where}: {text.get(ln, '')[:100]}")
