#!/bin/bash
for lib in paper_1008_1366_b200/libidconv.so $(ls tools/var_*.so 2>/dev/null); do
  echo "== $lib"
  for k in "cconv2d 1,1024,1024" "cconv2d 64,256,256" "hconv2d 4095,2048" "cconv3d 512,512,512" "hconv3d 1023,1023,512"; do
    IDCONV_LIB=$lib python tools/prof_nd.py $k --reps 2 | tail -1
  done
done
