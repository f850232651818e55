set -x
O=gpurun_out/r2reg; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -25 $O/pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 5 > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log | cut -c1-400
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 30 --warmup 5 > $O/bench_n2.log 2>&1; echo "bench2 rc $?"; tail -1 $O/bench_n2.log | cut -c1-600
