#!/bin/bash
# compute-sanitizer over scripts/sanitize_cases.py (on the GPU box); logs -> gpurun_out/
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
