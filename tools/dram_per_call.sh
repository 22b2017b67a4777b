#!/bin/bash
# DRAM bytes of one whole 3D call (every launch of the call, ncu, cold and
# serialised) -- the streaming traffic of the slab groups against B_alg
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for k in "cconv3d 512,512,512" "hconv3d 1023,1023,512"; do
  set -- $k
  python tools/prof_nd.py $1 $2 --reps 1 > /dev/null 2>&1 &&
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/dram_$1.csv python tools/prof_nd.py $1 $2 --reps 1 > /dev/null 2>&1
done
echo done
