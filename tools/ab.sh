#!/bin/bash
# A/B timing of library variants on the row kernels
for lib in paper_1008_1366_b200/libidconv.so $(ls tools/var_*.so 2>/dev/null); do
  echo "== $lib"
  for k in "hconv1d 4096 4096" "tconv1d 4096 4096" "cconv1d 1024 32768" "hconv1d 1024 32768" "cconv1d 512 65536" "hconv1d 512 65536" "cconv1d 256 131072" "hconv1d 2048 16384"; do
    IDCONV_LIB=$lib python tools/prof_rows.py $k --reps 3 | tail -1
  done
done
