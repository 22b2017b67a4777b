#!/bin/bash
for fr in ${FRACS:-1000 3000 10000 100000}; do
  echo "frac=$fr"
  IDC_SLAB_L2_FRAC=$fr python tools/prof_nd.py cconv3d 512,512,512 --reps 2 | tail -1
  IDC_SLAB_L2_FRAC=$fr python tools/prof_nd.py hconv3d 1023,1023,512 --reps 2 | tail -1
done
