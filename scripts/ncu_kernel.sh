#!/bin/bash
# One ncu --set full capture of the first launch matching REGEX in a command, with its SASS hot spots.
# Usage (on the box): bash scripts/ncu_kernel.sh TAG REGEX SKIP cmd...
TAG=$1; RE=$2; SKIP=$3; shift 3
mkdir -p gpurun_out /tmp/reps
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RE -s $SKIP -c 1 -f -o /tmp/reps/$TAG "$@" > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i /tmp/reps/$TAG.ncu-rep --page source --print-source sass --csv > /tmp/reps/${TAG}_src.csv 2>/dev/null
python scripts/sass_hot.py /tmp/reps/${TAG}_src.csv 50 > gpurun_out/${TAG}_sass_hot.txt 2>&1
ncu -i /tmp/reps/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/reps/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
