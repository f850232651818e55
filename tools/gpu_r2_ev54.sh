# W = 32 CTAs per channel (K=8: 256 CTAs, two per SM at 256 threads) vs 16
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for N in 2 4; do for S in 25000000 268435456; do for W in 16 32; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --ctas $W --bytes $S $FL > /tmp/o.log 2>&1; tail -1 /tmp/o.log | python -c "
import json,sys
l=sys.stdin.read()
try:
    d=json.loads(l); print('N=$N S=$S W=$W', round(d['ms_per_step']*1e3,1), 'us', round(d['busbw_per_rank'],1), d['config'].get('protocol', ''))
except Exception: print('N=$N S=$S W=$W failed'); import subprocess; print(open('/tmp/o.log').read()[-1500:])"
done; done; done
