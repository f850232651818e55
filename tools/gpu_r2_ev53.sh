# more CTAs per GPU: K=16 x W=16 (256 CTAs, 2 per SM) vs K=8 x W=16, 25 MB and 256 MiB
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for N in 2 4; do for S in 25000000 268435456; do for K in 8 16; do for P in AUTO; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --channels $K --ctas 16 --bytes $S --protocol $P $FL 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
    d=json.loads(l); print('N=$N S=$S K=$K', round(d['ms_per_step']*1e3,1), 'us', round(d['busbw_per_rank'],1))
except Exception: print('N=$N S=$S K=$K failed', l[:300])"
done; done; done; done
