IDCONV_LIB=tools/var_k3e16.so timeout 600 python -m pytest tests/test_parity_1d.py -m gpu -x -q -k "hconv or tconv" > gpurun_out/pt_k3e16.log 2>&1
bash tools/ab_all.sh > gpurun_out/ab_k3e16.log 2>&1
