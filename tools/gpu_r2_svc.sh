set -x
O=gpurun_out/r2svc; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_service.py -x -q -s > $O/pytest_service.log 2>&1; echo "service rc $?"
tail -15 $O/pytest_service.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -15 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"; tail -2 $O/smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.log 2>&1; echo "smoke-ncu rc $?"; tail -3 $O/smoke_ncu.log
timeout 300 python bench.py --steps 50 --warmup 5 > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log | cut -c1-600
