timeout 900 python -m pytest tests/test_parity_1d.py -m gpu -x -q > gpurun_out/pt_512w.log 2>&1
bash tools/ab_all.sh > gpurun_out/ab_512w.log 2>&1
timeout 900 python -m pytest tests/test_parity_nd.py -m gpu -x -q -k "3d" >> gpurun_out/pt_512w.log 2>&1
