"""Summarise an `ncu --page source --print-source sass --csv` dump: hottest instructions by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
iS, iI, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
num = lambda x: int(x) if x.strip().isdigit() else 0
tot = sum(num(r[iS]) for r in data)
totI = sum(num(r[iI]) for r in data)
print("samples", tot, "warp-instructions", totI)
from collections import Counter
op = Counter()
opi = Counter()
for r in data:
    m = r[iSrc].strip().split()[0] if r[iSrc].strip() else "?"
    if m.startswith("@"):
        m = r[iSrc].strip().split()[1]
    m = m.split(".")[0]
    op[m] += num(r[iS])
    opi[m] += num(r[iI])
print("by opcode (samples, inst):", [(k, v, opi[k]) for k, v in op.most_common(20)])
for r in sorted(data, key=lambda r: -num(r[iS]))[:n]:
    print(f"{num(r[iS]):6d} {num(r[iI]):9d}  {r[0][-5:]} {r[iSrc].strip()[:90]}")
