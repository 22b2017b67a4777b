#!/bin/bash
# A/B of library variants on the 3D/2D pencil configs only (tools/prof_nd.py)
for rep in 1 2; do
for lib in paper_1008_1366_b200/libidconv.so $(ls tools/var_*.so 2>/dev/null); do
  echo "== $lib"
  for k in "hconv2d 4095,2048" "hconv3d 1023,1023,512"; do
    IDCONV_LIB=$lib python tools/prof_nd.py $k --reps 4 | sort -t' ' -k4 -n | head -1
  done
done
done
