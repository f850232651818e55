set -x
O=gpurun_out/r2cc4; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_r2cc.py tests/test_gpu_service.py -x -q -s > $O/pytest_r2cc.log 2>&1; echo "r2cc rc $?"
tail -8 $O/pytest_r2cc.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -8 $O/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --steps 50 > $O/bench_n4.log 2>&1; echo "bench4 rc $?"
tail -1 $O/bench_n4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['busbw_per_rank']); print(json.dumps(d.get('r2cc_allreduce'))[:3000])"
