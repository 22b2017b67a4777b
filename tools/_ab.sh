bash tools/ab_all.sh > gpurun_out/ab_k3one.log 2>&1
timeout 900 python -m pytest tests/test_parity_1d.py tests/test_parity_nd.py -m gpu -x -q -k "hconv" > gpurun_out/pt_k3one.log 2>&1
IDCONV_LIB=tools/var_k8e8.so timeout 900 python -m pytest tests/test_parity_nd.py -m gpu -x -q -k "hconv and not config" > gpurun_out/pt_k8e8.log 2>&1
