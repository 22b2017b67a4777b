timeout 900 python -m pytest tests/test_parity_1d.py tests/test_dist.py -m gpu -x -q -k "cconv or dist or nccl or emulated" > gpurun_out/pt_k2one.log 2>&1
bash tools/ab_all.sh > gpurun_out/ab_k2one.log 2>&1
