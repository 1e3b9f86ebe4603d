#!/bin/bash
# ncu launch lists + full captures of the attention kernel for C3 (CogVideoX-like) and C4 (Llama GQA)
TAG=${1:-r02}
mkdir -p gpurun_out /tmp/reps gpurun_out/${TAG}_profiles
for cfg in c3_cogvideox c4_llama_gqa c2_4k_d128_causal; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_${cfg}.csv python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn -s 3 -c 1 -f -o /tmp/reps/${TAG}_prof_${cfg} python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python scripts/ncu_summary.py /tmp/reps/${TAG}_prof_${cfg}.ncu-rep gpurun_out/${TAG}_launches_${cfg}.csv $cfg ${TAG} > gpurun_out/${TAG}_summary_${cfg}.txt 2>&1
done
cp profiles/${TAG}_* profiles/traffic.json gpurun_out/${TAG}_profiles/ 2>/dev/null
echo done
