#!/bin/bash
# A/B: K2 row groups per CTA at m = 512 (IDC_K2_G512: in-tree 4, variants 5 / 6)
for rep in 1 2; do
for lib in paper_1008_1366_b200/libidconv.so $(ls tools/var_k2g*.so); do
  echo "== $lib"
  IDCONV_LIB=$lib python tools/prof_rows.py cconv1d 512 65536 --reps 9 | sort -t: -k2 -n | sed -n 5p
  IDCONV_LIB=$lib python tools/prof_nd.py cconv3d 512,512,512 --reps 3 | sort -t' ' -k4 -n | head -1
done
done
