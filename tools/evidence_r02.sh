#!/bin/bash
# round-2 evidence: the driver's commands (reference arm, default bench), then
# (EV_NCU=1) the ncu launch list of the headline-only bench command
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
t0=$SECONDS
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
echo "reference arm wall $((SECONDS - t0)) s" >> gpurun_out/ev_ref.err
t0=$SECONDS
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
echo "bench wall $((SECONDS - t0)) s" >> gpurun_out/ev_bench.err
if [ "${EV_NCU:-0}" = 1 ]; then
  CMD="python bench.py --parts= --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/ev_head_plain.json 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c5b.csv $CMD > gpurun_out/ev_ncu.log 2>&1
fi
echo done
