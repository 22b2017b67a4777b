python tools/prof_rows.py hconv1d 512 65536 --reps 1 > /dev/null 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:rows512w -c 1 -o gpurun_out/r02b_k3w -f python tools/prof_rows.py hconv1d 512 65536 --reps 1 > gpurun_out/r02b_k3w.log 2>&1
