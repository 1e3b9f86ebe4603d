#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + one full capture of the attention kernel.
# Usage (on the box): bash scripts/gpu_round.sh [tests|bench|ncu|all] [bench-config]
set -u
mkdir -p gpurun_out
what=${1:-all}
cfg=${2:-c2_32k_d128}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
if [[ $what == all || $what == tests ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
if [[ $what == all || $what == bench ]]; then
  timeout 900 python bench.py --config $cfg > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
fi
if [[ $what == all || $what == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
      python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_attn -s 3 -c 1 -f -o gpurun_out/prof_attn_$cfg \
      python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none -k 'regex:k_kv_stats|k_kv_quant|k_q_quant|k_delta_s' -s 4 -c 4 -f \
      -o gpurun_out/prof_prep_$cfg python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/ncu_prep.log 2>&1
fi
echo done
