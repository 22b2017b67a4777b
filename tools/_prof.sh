python tools/prof_nd.py hconv3d 1023,1023,512 --reps 1 > /dev/null 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:pad0_bwd_warp -c 1 -o gpurun_out/r02c_k7w -f python tools/prof_nd.py hconv3d 1023,1023,512 --reps 1 > gpurun_out/r02c_k7w.log 2>&1
