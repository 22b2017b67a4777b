#!/bin/bash
# ncu --set full of the dominant 2D/3D kernels (first launch of each), reports in gpurun_out/
mkdir -p gpurun_out
t=${1:-r01nd}
bash tools/prof_pencil.sh ${t}_c4_rows hconv2d 4095,2048 hconv_rows3
bash tools/prof_pencil.sh ${t}_c4_k7 hconv2d 4095,2048 pad0_bwd
bash tools/prof_pencil.sh ${t}_c4_k8 hconv2d 4095,2048 pad0_fwd
bash tools/prof_pencil.sh ${t}_c5a_k5x cconv3d 512,512,512 pad_bwd
bash tools/prof_pencil.sh ${t}_c5a_rows cconv3d 512,512,512 cconv_rows
bash tools/prof_pencil.sh ${t}_c5b_k7x hconv3d 1023,1023,512 pad0_bwd
bash tools/prof_pencil.sh ${t}_c5b_rows hconv3d 1023,1023,512 hconv_rows3
bash tools/prof_pencil.sh ${t}_c4t_k5 tconv2d 4096,2048 pad_bwd
bash tools/prof_pencil.sh ${t}_c4t_rows tconv2d 4096,2048 tconv_rows3
bash tools/prof_pencil.sh ${t}_c3a_k5 cconv2d 1,1024,1024 pad_bwd
bash tools/prof_pencil.sh ${t}_c3a_rows cconv2d 1,1024,1024 cconv_rows
