FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for i in 1 2; do
for N in 2 4; do
for C in 262144 524288 1048576 2097152 4194304; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --chunk $C $FL 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=$N chunk $C', round(d['ms_per_step'],4), round(d['busbw_per_rank'],1))"
done; done; done
for N in 2 4; do for C in 524288 1048576; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --chunk $C --bytes 1073741824 $FL 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=$N 1GiB chunk $C', round(d['ms_per_step'],4), round(d['busbw_per_rank'],1))"
done; done
