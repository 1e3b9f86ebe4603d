"""Summarise ncu output for profiles/ (run here, on the CPU side, after a gpurun call).

    python scripts/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv CONFIG TAG

Writes profiles/<TAG>_ncu_<kernel>_<CONFIG>_metrics.json (key metrics of the captured attention
kernel), profiles/<TAG>_launches_<CONFIG>.csv (our kernels' per-launch durations from the
`--metrics gpu__time_duration.sum` pass) and updates profiles/traffic.json (DRAM bytes per launch,
read by bench.py's roofline.traffic).  Prints the per-kernel share of the step."""
import csv
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio")


def main():
    rep, launches, cfg, tag = sys.argv[1:5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"Kernel Name": [vals[hdr.index("Kernel Name")], ""]}
    for k in KEEP:
        if k in hdr:
            i = hdr.index(k)
            out[k] = [vals[i], units[i]]
    kname = re.search(r"(k_\w+)<", out["Kernel Name"][0]).group(1)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{kname}_{cfg}_metrics.json"), "w") as f:
        json.dump(out, f, indent=1)

    def gb(key):
        v, u = out[key]
        return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[u]
    traffic = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
    tj[cfg] = {"kernel": out["Kernel Name"][0], "dram_bytes_per_launch": traffic,
               "source": f"profiles/{tag}_ncu_{kname}_{cfg}_metrics.json"}
    json.dump(tj, open(tpath, "w"), indent=1)

    # launch list: keep our kernels only (sage2 namespace), drop torch's input generation
    per = defaultdict(list)
    lines = [l for l in open(launches) if l.startswith('"')]
    rd = list(csv.reader(lines))
    h = rd[0]
    ours = []
    for r in rd[1:]:
        name = r[h.index("Kernel Name")]
        if "sage2" not in name and not re.search(r"\bk_\w+<", name):
            continue
        dur = float(r[h.index("Metric Value")])
        unit = r[h.index("Metric Unit")]
        dur_ms = dur * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        short = re.search(r"(k_\w+<[^>]*>)", name)
        short = short.group(1) if short else name[:60]
        per[short].append(dur_ms)
        ours.append((short, dur_ms))
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches_{cfg}.csv"), "w") as f:
        f.write("kernel,ms\n")
        for k, ms in ours:
            f.write(f"{k},{ms:.6f}\n")
    tot = sum(ms for _, ms in ours)
    print(f"{cfg}: DRAM traffic of {kname} = {traffic / 1e9:.3f} GB/launch")
    for k, v in per.items():
        avg = sum(v) / len(v)
        print(f"  {k:40s} {len(v):3d} launches  {avg:9.3f} ms/launch  share {sum(v) / tot:6.1%}")


if __name__ == "__main__":
    main()
