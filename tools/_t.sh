timeout 900 python -m pytest tests/test_transform_counts.py tests/test_guard_regions.py -m gpu -q > gpurun_out/pt_new.log 2>&1
