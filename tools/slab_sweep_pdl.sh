for cfg in "2 2000" "2 1000" "2 4000" "3 2000" "3 1000" "4 1000" "2 2000"; do
  set -- $cfg
  echo "streams=$1 frac=$2"
  IDC_SLAB_STREAMS=$1 IDC_SLAB_L2_FRAC=$2 python tools/prof_nd.py cconv3d 512,512,512 --reps 3 | sort -t' ' -k4 -n | head -1
  IDC_SLAB_STREAMS=$1 IDC_SLAB_L2_FRAC=$2 python tools/prof_nd.py hconv3d 1023,1023,512 --reps 3 | sort -t' ' -k4 -n | head -1
done
