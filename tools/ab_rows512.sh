#!/bin/bash
# A/B of library variants on the m = 512 row kernels and the 3D configs
for rep in 1 2; do
for lib in paper_1008_1366_b200/libidconv.so $(ls tools/var_*.so 2>/dev/null); do
  echo "== $lib"
  for k in "hconv1d 512 65536" "cconv1d 512 65536"; do
    IDCONV_LIB=$lib python tools/prof_rows.py $k --reps 5 | tail -1
  done
  for k in "cconv3d 512,512,512" "hconv3d 1023,1023,512"; do
    IDCONV_LIB=$lib python tools/prof_nd.py $k --reps 4 | sort -t' ' -k4 -n | head -1
  done
done
done
