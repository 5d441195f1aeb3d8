"""Average the FV_JPEG_TIMING phase lines of a log (skipping the first N calls):
    FV_JPEG_TIMING=1 python bench.py --ops jpeg ... 2> log; python tools/jpeg_phase_avg.py log [skip]"""
import collections
import re
import sys

skip = int(sys.argv[2]) if len(sys.argv) > 2 else 5
calls, cur = [], collections.OrderedDict()
for line in open(sys.argv[1]):
    m = re.match(r"\[fv_jpeg_gpu\]\s+(gpu )?(.*?)\s+([0-9.]+) ms$", line.rstrip())
    if not m:
        continue
    key = ("gpu " if m.group(1) else "") + m.group(2)
    if key == "parse + plan" and cur:
        calls.append(cur)
        cur = collections.OrderedDict()
    cur.setdefault(key, 0.0)
    cur[key] += float(m.group(3))
if cur:
    calls.append(cur)
use = calls[skip:]
print(f"{len(calls)} calls, averaging {len(use)}")
for k in use[0]:
    v = [c.get(k, 0.0) for c in use]
    print(f"  {k:34s} mean {sum(v)/len(v):7.3f}  min {min(v):7.3f}  max {max(v):7.3f}")
