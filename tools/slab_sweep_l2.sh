#!/bin/bash
# slab groups at and below L2 size (IDC_SLAB_L2_FRAC = percent of L2 per set of groups in flight)
for cfg in "2 2000" "4 50" "4 100" "2 50" "2 100" "4 200" "2 400" "4 25"; do
  set -- $cfg
  echo "streams=$1 frac=$2"
  IDC_SLAB_STREAMS=$1 IDC_SLAB_L2_FRAC=$2 python tools/prof_nd.py cconv3d 512,512,512 --reps 3 | tail -1
  IDC_SLAB_STREAMS=$1 IDC_SLAB_L2_FRAC=$2 python tools/prof_nd.py hconv3d 1023,1023,512 --reps 3 | tail -1
done
