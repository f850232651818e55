set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_gpu.log
for i in 1 2; do R2_DEBUG=1 BYTES=268435456 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 tools/debug_multi.py > gpurun_out/dbg4_$i.log 2>&1; echo "dbg rc $?"; grep "faulted call" gpurun_out/dbg4_$i.log; done
timeout 300 python bench.py > gpurun_out/bench1.log 2>&1; echo "bench1 rc $?"; tail -1 gpurun_out/bench1.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 4 > gpurun_out/bench4.log 2>&1; echo "bench4 rc $?"; tail -1 gpurun_out/bench4.log
