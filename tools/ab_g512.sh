#!/bin/bash
# A/B: K3 row groups per CTA at m <= 512 (IDC_K3_G512: in-tree 6, variants 4 / 5)
for rep in 1 2; do
for lib in paper_1008_1366_b200/libidconv.so $(ls tools/var_k3g*.so); do
  echo "== $lib"
  IDCONV_LIB=$lib python tools/prof_rows.py hconv1d 512 65536 --reps 9 | sort -t: -k2 -n | sed -n 5p
  IDCONV_LIB=$lib python tools/prof_nd.py hconv3d 1023,1023,512 --reps 3 | sort -t' ' -k4 -n | head -1
  IDCONV_LIB=$lib python tools/prof_nd.py hconv2d 1023,512 --reps 5 | sort -t' ' -k4 -n | head -1
done
done
