FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for i in 1 2; do
for N in 4 2; do
for T in 256 320 384 512; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --threads $T $FL 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=$N threads $T', round(d['ms_per_step'],4), round(d['busbw_per_rank'],1))"
done; done; done
