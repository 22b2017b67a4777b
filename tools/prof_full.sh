#!/bin/bash
# ncu --set full captures of the dominant kernels (one launch each), reports in gpurun_out/
mkdir -p gpurun_out
tag=${1:-x}
python tools/prof_rows.py cconv1d 1024 32768 --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:_rows -c 1 -o gpurun_out/${tag}_cconv1024 -f \
    python tools/prof_rows.py cconv1d 1024 32768 --reps 1 > gpurun_out/${tag}_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:_rows -c 1 -o gpurun_out/${tag}_hconv4096 -f \
    python tools/prof_rows.py hconv1d 4096 4096 --reps 1 >> gpurun_out/${tag}_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:_rows -c 1 -o gpurun_out/${tag}_tconv4096 -f \
    python tools/prof_rows.py tconv1d 4096 4096 --reps 1 >> gpurun_out/${tag}_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pad0_bwd -c 1 -o gpurun_out/${tag}_pad0bwd2048 -f \
    python tools/prof_nd.py hconv2d 4095,2048 --reps 1 >> gpurun_out/${tag}_ncu.log 2>&1
