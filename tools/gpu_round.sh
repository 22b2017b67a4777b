#!/bin/bash
# One GPU session of round evidence ($1 = tag, default r01):
#   pytest -m gpu, smoke, bench lines for every workload + the reference arm,
#   the ncu launch list of the default bench command, and ncu --set full
#   captures of the dominant kernels (DRAM bytes per launch).
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "exit=$?" >> gpurun_out/${tag}_pytest_gpu.log
python __graft_entry__.py --smoke > gpurun_out/${tag}_smoke.log 2>&1
bash tools/bench_all.sh $tag
python bench.py --impl reference --steps 2 --warmup 1 --cpu-budget 20 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"_rows|pad" --csv --log-file gpurun_out/${tag}_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${tag}_ncu_launches.log 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launches_c2.csv > gpurun_out/${tag}_launches_c2_summary.txt 2>&1
bash tools/prof_one.sh ${tag}_prof_tconv tconv1d 4096 4096
bash tools/prof_one.sh ${tag}_prof_hconv hconv1d 4096 4096
bash tools/prof_one.sh ${tag}_prof_cconv cconv1d 1024 32768
ls gpurun_out | grep $tag
