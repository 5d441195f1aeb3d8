"""Aggregate an ncu report's SASS instruction counts by CUDA source line:
    python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Instructions Executed" in r)
ei = hdr.index("Instructions Executed")
agg = collections.Counter()
text = {}
cur = None
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= ei:
        continue
    if r[0]:
        cur = int(r[0]) if r[0].isdigit() else cur
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
    print(f"{100 * n / tot:5.1f}% {n:>12d}  {ln}: {text.get(ln, '')[:100]}")
