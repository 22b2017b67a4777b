#!/bin/bash
# ncu --set full of the dominant kernel of every bench config (first launch),
# reports in gpurun_out/r02p_*.ncu-rep (per-unit DRAM traffic: tools/traffic_from_ncu.py)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
prof() {  # tag regex command...
  local tag=$1 re=$2; shift 2
  "$@" > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:$re -c 1 \
      -o gpurun_out/r02p_$tag -f "$@" > gpurun_out/r02p_$tag.log 2>&1
}
prof c1_k2 cconv_rows2 python tools/prof_rows.py cconv1d 1024 32768 --reps 1
prof c2a_k3 hconv_rows3 python tools/prof_rows.py hconv1d 4096 4096 --reps 1
prof c2b_k4 tconv_rows3 python tools/prof_rows.py tconv1d 4096 4096 --reps 1
prof c3a_k2 cconv_rows2 python tools/prof_nd.py cconv2d 1,1024,1024 --reps 1
prof c3b_k2 cconv_rows2 python tools/prof_nd.py cconv2d 64,256,256 --reps 1
prof c4_k3 hconv_rows3 python tools/prof_nd.py hconv2d 4095,2048 --reps 1
prof c5a_k2 cconv_rows2 python tools/prof_nd.py cconv3d 512,512,512 --reps 1
prof c5a_k5 pad_bwd_tma python tools/prof_nd.py cconv3d 512,512,512 --reps 1
prof c5b_k3 hconv_rows3 python tools/prof_nd.py hconv3d 1023,1023,512 --reps 1
prof c5b_k7 pad0_bwd_tma python tools/prof_nd.py hconv3d 1023,1023,512 --reps 1
# keep only text: ncu summaries and raw metric CSVs (the reports exceed the copy-back limit)
for r in gpurun_out/r02p_*.ncu-rep; do
  python tools/ncu_summary.py "$r" > "${r%.ncu-rep}.txt" 2>&1
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  rm -f "$r"
done
echo done
