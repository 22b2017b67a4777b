#!/bin/bash
# ncu --set full of one row-kernel launch: prof_one.sh <tag> <kind> <m> <batch>
mkdir -p gpurun_out
python tools/prof_rows.py $2 $3 $4 --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:_rows -c 1 -o gpurun_out/$1 -f \
    python tools/prof_rows.py $2 $3 $4 --reps 1 > gpurun_out/$1.log 2>&1
