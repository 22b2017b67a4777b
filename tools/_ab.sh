timeout 900 python -m pytest tests/test_parity_nd.py tests/test_guard_regions.py -m gpu -x -q -k "hconv" > gpurun_out/pt_k7w.log 2>&1 && bash tools/ab_all.sh > gpurun_out/ab_k7w.log 2>&1
