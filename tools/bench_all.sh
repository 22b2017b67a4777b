#!/bin/bash
# bench lines for every workload (round evidence); $1 = tag
tag=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${tag}_smi.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err
for w in c1 c3a c3b c4 c4adv c4t c5a c5b; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
