#!/bin/bash
# slab-group sweep after the pencil changes (streams, % of L2 per group set)
for cfg in "2 2000" "2 4000" "2 8000" "1 4000" "3 2000" "2 1000"; do
  set -- $cfg
  echo "streams=$1 frac=$2"
  IDC_SLAB_STREAMS=$1 IDC_SLAB_L2_FRAC=$2 python tools/prof_nd.py cconv3d 512,512,512 --reps 2 | tail -1
  IDC_SLAB_STREAMS=$1 IDC_SLAB_L2_FRAC=$2 python tools/prof_nd.py hconv3d 1023,1023,512 --reps 2 | tail -1
done
