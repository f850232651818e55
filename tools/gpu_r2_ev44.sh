for N in 4; do
SIZES=1024,65536 R2_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N tools/trace_multi.py 2>&1 | grep rank
SIZES=1024 R2_TRACE=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N tools/trace_multi.py 2>&1 | grep rank
R2_DEBUG=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N tools/host_overhead.py 2>&1 | grep -v "^\*\|OMP"
done
