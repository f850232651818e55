timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rs 2>&1 | tail -4
