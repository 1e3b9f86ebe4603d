#!/bin/bash
# Bench lines for several BASELINE configs (kernel-only numbers are in roofline.achieved).
mkdir -p gpurun_out
for cfg in "$@"; do
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/sweep_$cfg.json 2> gpurun_out/sweep_$cfg.err
  python - "$cfg" <<'PY'
import json,sys
cfg=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/sweep_{cfg}.json").read().strip().splitlines()[-1])
    print(f"{cfg:22s} step {d['value']:8.1f} TOPS  ms {d['ms_per_step']:8.2f}  kernel {d['roofline']['achieved']:8.1f} TOPS ({d['roofline']['kernel_ms']:.2f} ms, frac {d['roofline']['frac']:.3f})  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(cfg, "FAILED", e, open(f"gpurun_out/sweep_{cfg}.err").read()[-500:])
PY
done
