#!/bin/bash
# prepare() A/B over the C2 / C3 / C4 shapes between library builds: bash scripts/prep_sweep.sh LIB1,LIB2
L=$1
for n in 1024 2048 4096 16384 32768; do python scripts/prep_ab2.py $L 4 32 32 $n 128; done
python scripts/prep_ab2.py $L 4 32 32 1024 64
python scripts/prep_ab2.py $L 4 32 32 4096 128 1
python scripts/prep_ab2.py $L 1 48 48 17776 64
python scripts/prep_ab2.py $L 1 32 8 100000 128 1
