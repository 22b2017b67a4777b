timeout 900 python -m pytest tests/test_dist.py tests/test_parity_nd.py -m gpu -x -q -k "dist or emulated or nccl or tma or tall" > gpurun_out/pt_dist2.log 2>&1
timeout 600 python tools/dist_p1_bench.py > gpurun_out/dist_p1.log 2>&1
