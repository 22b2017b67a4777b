#!/bin/bash
# ncu --set full of the first K7 and K8 launches (fft0pad pencils at m = 512) of one C5b call
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
t=${1:-r02}
python tools/prof_nd.py hconv3d 1023,1023,512 --reps 1 > gpurun_out/${t}_plain.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:pad0_bwd_tma -c 1 -o gpurun_out/${t}_k7 -f \
    python tools/prof_nd.py hconv3d 1023,1023,512 --reps 1 > gpurun_out/${t}_ncu_k7.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pad0_fwd_tma -c 1 -o gpurun_out/${t}_k8 -f \
    python tools/prof_nd.py hconv3d 1023,1023,512 --reps 1 > gpurun_out/${t}_ncu_k8.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:hconv_rows3 -c 1 -o gpurun_out/${t}_k3 -f \
    python tools/prof_nd.py hconv3d 1023,1023,512 --reps 1 > gpurun_out/${t}_ncu_k3.log 2>&1
