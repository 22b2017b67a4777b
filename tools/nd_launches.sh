#!/bin/bash
# Per-kernel time breakdown (ncu launch lists) of one call of every ND config.
mkdir -p gpurun_out
for k in "cconv2d 1,1024,1024 c3a" "cconv2d 64,256,256 c3b" "hconv2d 4095,2048 c4" "tconv2d 4096,2048 c4t" "cconv3d 512,512,512 c5a" "hconv3d 1023,1023,512 c5b"; do
  set -- $k
  python tools/prof_nd.py $1 $2 --reps 2 > gpurun_out/nd_$3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"_rows|pad" --csv --log-file gpurun_out/launches_$3.csv \
      python tools/prof_nd.py $1 $2 --reps 1 >> gpurun_out/nd_$3.log 2>&1
  python tools/launch_summary.py gpurun_out/launches_$3.csv > gpurun_out/launches_$3_summary.txt 2>&1
done
