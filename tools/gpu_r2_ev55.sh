# W = 32 (two CTAs per SM) with every protocol at 256 threads, vs W = 16
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for N in 2 4; do for S in 25000000 268435456 67108864; do for cfg in "16 0" "16 256" "32 256"; do
set -- $cfg; W=$1; LT=$2
if [ $LT = 0 ]; then unset R2_LL_THREADS; else export R2_LL_THREADS=$LT; fi
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --ctas $W --bytes $S $FL > /tmp/o.log 2>&1; tail -1 /tmp/o.log | python -c "
import json,sys
l=sys.stdin.read()
try:
    d=json.loads(l); print('N=$N S=$S W=$W llthreads=$LT', round(d['ms_per_step']*1e3,1), 'us', round(d['busbw_per_rank'],1))
except Exception: print('N=$N S=$S W=$W llthreads=$LT failed'); print([x for x in open('/tmp/o.log').read().splitlines() if 'Error' in x][:3])"
done; done; done
