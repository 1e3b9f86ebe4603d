"""Per-kernel HBM summary of an `ncu --set full` capture of the preprocessing kernels.

    python scripts/ncu_prep_summary.py REPORT.ncu-rep OUT.json

For each captured launch: duration, DRAM bytes read / written, achieved GB/s and its fraction of the
measured copy bandwidth in MEASURED_PEAKS.json (hbm_gbs)."""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "msecond": 1e-3, "us": 1e-6,
         "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}


def main():
    rep, out_path = sys.argv[1:3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    res = []
    for vals in rows[2:]:
        if len(vals) != len(hdr):
            continue
        def get(k):
            i = hdr.index(k)
            return float(vals[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        t = get("gpu__time_duration.sum")
        rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        name = re.search(r"(k_\w+<[^>]*>)", vals[hdr.index("Kernel Name")])
        res.append({"kernel": name.group(1) if name else vals[hdr.index("Kernel Name")][:60],
                    "ms": t * 1e3, "dram_read_GB": rd / 1e9, "dram_write_GB": wr / 1e9,
                    "dram_GBps": (rd + wr) / t / 1e9, "frac_of_measured_hbm": (rd + wr) / t / 1e9 / peak})
    json.dump(res, open(out_path, "w"), indent=1)
    for r in res:
        print(f"{r['kernel']:28s} {r['ms']:7.3f} ms  {r['dram_read_GB']:6.3f} + {r['dram_write_GB']:6.3f} GB  "
              f"{r['dram_GBps']:7.0f} GB/s = {r['frac_of_measured_hbm']:.2f} of {peak}")


if __name__ == "__main__":
    main()
