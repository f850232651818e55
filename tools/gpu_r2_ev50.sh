# round-1 kernel (commit 8b054b2, built in _r1tree) vs HEAD on one box: 256 MiB bf16 headline, N=2 / N=4, 512 KiB chunks
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10 --chunk 524288"
for rep in 1 2; do
for T in _r1tree .; do
for N in 2 4; do
(cd $T && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N $FL 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tree $T N=$N', round(d['ms_per_step'],4), round(d['busbw_per_rank'],1))")
done; done; done
