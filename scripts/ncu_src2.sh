#!/bin/bash
# ncu source-view capture of one attention launch (kernel_ab.py), SASS csv gzipped into gpurun_out/
TAG=$1; RE=$2; shift 2
mkdir -p gpurun_out /tmp/reps
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RE -s 2 -c 1 -f -o /tmp/reps/$TAG "$@" > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i /tmp/reps/$TAG.ncu-rep --page source --print-source sass --csv 2>/dev/null | gzip -c > gpurun_out/${TAG}_src.csv.gz
