mkdir -p gpurun_out
for rep in 1 2; do
for lib in paper_1008_1366_b200/libidconv.so tools/var_k4s0.so tools/var_k4s2048.so; do
  echo "== $lib"
  for k in "tconv1d 4096 4096" "tconv1d 2048 8192" "tconv1d 1024 16384"; do
    IDCONV_LIB=$lib python tools/prof_rows.py $k --reps 9 | sort -t: -k2 -n | sed -n 5p
  done
  IDCONV_LIB=$lib python tools/prof_nd.py tconv2d 4096,2048 --reps 5 | sort -t' ' -k4 -n | head -1
done
done
