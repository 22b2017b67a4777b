#!/bin/bash
# ncu --set full of the first (full-array x-pass) launch of a pencil kernel
mkdir -p gpurun_out
tag=$1; kind=$2; shape=$3; regex=$4
python tools/prof_nd.py $kind $shape --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:$regex -c 1 -o gpurun_out/$tag -f \
    python tools/prof_nd.py $kind $shape --reps 1 > gpurun_out/$tag.log 2>&1
