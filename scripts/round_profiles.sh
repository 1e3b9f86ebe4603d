#!/bin/bash
# Round-end evidence in one gpurun call: bench line, reference arm, full sweep, ncu launch lists,
# full ncu captures of the attention kernels (d=128 v8, d=64 v12) and of the preprocessing kernels.
# Usage (on the box): bash scripts/round_profiles.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out /tmp/reps gpurun_out/${TAG}_profiles
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
bash scripts/bench_sweep.sh c1_256_d64 c2_1k_d64 c2_1k_d64_causal c2_1k_d128 c2_1k_d128_causal c2_4k_d64 c2_4k_d64_causal c2_4k_d128 c2_4k_d128_causal c2_16k_d64 c2_16k_d64_causal c2_16k_d128 c2_16k_d128_causal c2_32k_d64 c2_32k_d64_causal c2_32k_d128 c2_32k_d128_causal c3_cogvideox c4_llama_gqa c5_b8 > gpurun_out/${TAG}_sweep.txt 2>&1
for cfg in c2_32k_d128 c2_4k_d128 c2_32k_d64; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_${cfg}.csv python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn8 -s 3 -c 1 -f -o /tmp/reps/${TAG}_prof_attn8_c2_32k_d128 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn12 -s 3 -c 1 -f -o /tmp/reps/${TAG}_prof_attn12_c2_32k_d64 python bench.py --config c2_32k_d64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k 'regex:k_kv_stats|k_kv_quant|k_q_quant|k_delta_s' -s 5 -c 5 -f -o /tmp/reps/${TAG}_prof_prep_c2_32k_d128 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# summaries only (the .ncu-rep files stay on the box: gpurun returns <= 64 MiB)
python scripts/ncu_summary.py /tmp/reps/${TAG}_prof_attn8_c2_32k_d128.ncu-rep gpurun_out/${TAG}_launches_c2_32k_d128.csv c2_32k_d128 ${TAG} > gpurun_out/${TAG}_summary_32k.txt 2>&1
python scripts/ncu_summary.py /tmp/reps/${TAG}_prof_attn12_c2_32k_d64.ncu-rep gpurun_out/${TAG}_launches_c2_32k_d64.csv c2_32k_d64 ${TAG} > gpurun_out/${TAG}_summary_32k_d64.txt 2>&1
python scripts/ncu_prep_summary.py /tmp/reps/${TAG}_prof_prep_c2_32k_d128.ncu-rep profiles/${TAG}_ncu_prep_c2_32k_d128.json > gpurun_out/${TAG}_summary_prep.txt 2>&1
ncu -i /tmp/reps/${TAG}_prof_attn8_c2_32k_d128.ncu-rep --page source --print-source sass --csv > /tmp/reps/src8.csv 2>/dev/null
python scripts/sass_hot.py /tmp/reps/src8.csv 40 > gpurun_out/${TAG}_sass_hot_attn8.txt 2>&1
ncu -i /tmp/reps/${TAG}_prof_attn12_c2_32k_d64.ncu-rep --page source --print-source sass --csv > /tmp/reps/src12.csv 2>/dev/null
python scripts/sass_hot.py /tmp/reps/src12.csv 40 > gpurun_out/${TAG}_sass_hot_attn12.txt 2>&1
cp profiles/${TAG}_* profiles/traffic.json gpurun_out/${TAG}_profiles/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
echo done
