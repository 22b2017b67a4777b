timeout 600 python -m pytest tests/test_concurrency.py tests/test_abi.py -m gpu -q > gpurun_out/pt_conc.log 2>&1
timeout 1200 python tools/cufft_explicit.py > gpurun_out/cufft_r02.log 2>&1
