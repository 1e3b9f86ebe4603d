#!/bin/bash
# One ncu --set full capture of an attention kernel (kernel_ab.py launch) + its SASS source page.
# Usage (on the box): bash scripts/ncu_src.sh TAG N d variant [B H]
TAG=$1; N=$2; d=$3; VAR=$4; B=${5:-4}; H=${6:-32}
mkdir -p gpurun_out /tmp/reps
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn -s 2 -c 1 -f -o /tmp/reps/$TAG \
    python scripts/kernel_ab.py $N $d $VAR 1 $B $H > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i /tmp/reps/$TAG.ncu-rep --page source --print-source sass --csv > /tmp/reps/${TAG}_src.csv 2>/dev/null
python scripts/sass_hot.py /tmp/reps/${TAG}_src.csv 60 > gpurun_out/${TAG}_sass_hot.txt 2>&1
ncu -i /tmp/reps/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
gzip -c /tmp/reps/${TAG}_src.csv > gpurun_out/${TAG}_src.csv.gz
