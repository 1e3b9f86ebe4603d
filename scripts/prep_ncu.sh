#!/bin/bash
# per-kernel duration and DRAM bytes of sage2_prepare (ncu, one library): bash scripts/prep_ncu.sh TAG LIB B Hq Hkv N d
TAG=$1; shift; LIB=$1; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/${TAG}.csv python scripts/prep_ab2.py $LIB "$@" > /dev/null 2>&1
python - gpurun_out/${TAG}.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
iid = h.index("ID")
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault((r[iid], r[iK][:28]), {})[r[iM]] = float(r[iV].replace(",", ""))
agg = collections.OrderedDict()
for (i, k), m in per.items():
    agg.setdefault(k, []).append(m)
for k, ms in agg.items():
    n = len(ms); f = lambda key: sum(m.get(key, 0) for m in ms) / n
    t = f("gpu__time_duration.sum"); rd = f("dram__bytes_read.sum"); wr = f("dram__bytes_write.sum")
    print(f"{k:28s} n={n:3d} {t/1e3:8.1f} us  rd {rd/1e6:8.1f} MB wr {wr/1e6:8.1f} MB  {(rd+wr)/t:6.0f} GB/s  sm% {f('sm__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f} occ% {f('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} grid {f('launch__grid_size'):7.0f} regs {f('launch__registers_per_thread'):4.0f}")
PY
