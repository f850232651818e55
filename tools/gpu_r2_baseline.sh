set -x
mkdir -p gpurun_out/r2base
O=gpurun_out/r2base
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -5 $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 > $O/bench_n2.log 2>&1; echo "bench2 rc $?"; tail -1 $O/bench_n2.log
