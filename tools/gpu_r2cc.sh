set -x
O=gpurun_out/r2cc; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_r2cc.py tests/test_gpu_service.py -x -q -s > $O/pytest_r2cc.log 2>&1; echo "r2cc rc $?"
tail -30 $O/pytest_r2cc.log
