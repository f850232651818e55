set -x
O=gpurun_out/ev22; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --no-e2e --no-coll --no-fault > $O/bench_n4.log 2>&1; echo "bench4 rc $?"; tail -1 $O/bench_n4.log | cut -c1-400
