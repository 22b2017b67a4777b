#!/bin/bash
for cfg in "4 1000" "4 500" "4 2000" "2 1000" "2 2000" "3 1000"; do
  set -- $cfg
  echo "streams=$1 frac=$2"
  IDC_SLAB_STREAMS=$1 IDC_SLAB_L2_FRAC=$2 python tools/prof_nd.py cconv3d 512,512,512 --reps 2 | tail -1
  IDC_SLAB_STREAMS=$1 IDC_SLAB_L2_FRAC=$2 python tools/prof_nd.py hconv3d 1023,1023,512 --reps 2 | tail -1
done
