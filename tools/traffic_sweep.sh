#!/bin/bash
# one ncu --set full pass over every launch of one call per 2D config (tools/traffic_sweep.py)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/traffic_sweep.py units > gpurun_out/traffic_units.json 2> gpurun_out/traffic_units.err &&
python tools/traffic_sweep.py run > gpurun_out/traffic_plain.log 2>&1 &&
ncu --set full --clock-control none -k regex:'^k_|::k_' -o gpurun_out/traffic_sweep -f \
    python tools/traffic_sweep.py run > gpurun_out/traffic_ncu.log 2>&1
ncu -i gpurun_out/traffic_sweep.ncu-rep --page raw --csv > gpurun_out/traffic_sweep.raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/traffic_sweep.ncu-rep > gpurun_out/traffic_sweep.txt 2>&1
rm -f gpurun_out/traffic_sweep.ncu-rep
echo done
