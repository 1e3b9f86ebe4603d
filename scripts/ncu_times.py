"""Print median per-kernel durations from an `ncu --metrics gpu__time_duration.sum --csv` log.
    python scripts/ncu_times.py LOG [name-regex]"""
import csv
import re
import statistics
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rd = list(csv.reader(lines))
h = rd[0]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
d = defaultdict(list)
for r in rd[1:]:
    if len(r) != len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    n = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    if pat and not pat.search(n):
        continue
    unit = r[h.index("Metric Unit")]
    v = float(r[h.index("Metric Value")]) * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    d[n].append(v)
for n, v in d.items():
    print(f"{n[:50]:50s} n={len(v):3d} median {statistics.median(v):9.1f} us")
