#!/bin/bash
# A/B timing of library variants (in-tree lib + tools/var_*.so) on the
# config-size calls: 1D rows (tools/prof_rows.py) and 2D/3D (tools/prof_nd.py)
for lib in paper_1008_1366_b200/libidconv.so $(ls tools/var_*.so 2>/dev/null); do
  echo "== $lib"
  for k in "hconv1d 4096 4096" "tconv1d 4096 4096" "cconv1d 1024 32768" "hconv1d 512 65536" "cconv1d 512 65536"; do
    IDCONV_LIB=$lib python tools/prof_rows.py $k --reps 5 | tail -1
  done
  for k in "cconv2d 1,1024,1024" "cconv2d 64,256,256" "hconv2d 4095,2048" "cconv3d 512,512,512" "hconv3d 1023,1023,512"; do
    IDCONV_LIB=$lib python tools/prof_nd.py $k --reps 4 | sort -t' ' -k4 -n | head -1
  done
done
