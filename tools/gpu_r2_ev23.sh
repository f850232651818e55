for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_service.py -q -s 2>&1 | grep -E "failover under|passed|failed"; done
