#!/bin/bash
# One GPU session of evidence: default bench line, every workload, ncu launch
# list of the default bench command (our kernels), full captures of the
# dominant kernels (dram bytes per launch -> profiles/traffic.json).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3a c3b c4 c5a c5b; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
python bench.py --impl reference --steps 2 --warmup 1 --cpu-budget 20 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"_rows|pad" --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launches.log 2>&1
python tools/prof_rows.py tconv1d 4096 4096 --reps 1 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:_rows -c 1 -o gpurun_out/prof_tconv \
    python tools/prof_rows.py tconv1d 4096 4096 --reps 1 > gpurun_out/ncu_full.log 2>&1
python tools/prof_rows.py hconv1d 4096 4096 --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:_rows -c 1 -o gpurun_out/prof_hconv \
    python tools/prof_rows.py hconv1d 4096 4096 --reps 1 >> gpurun_out/ncu_full.log 2>&1
ls gpurun_out
