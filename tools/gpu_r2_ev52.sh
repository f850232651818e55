# N=2 / N=4 25 MB bucket: protocol x CTAs per channel
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 200 --warmup 10 --bytes 25000000"
for N in 2 4; do for P in SIMPLE LL128; do for W in 4 8 16; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --protocol $P --ctas $W $FL 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N=$N $P W=$W', round(d['ms_per_step']*1e3,1), 'us', round(d['busbw_per_rank'],1))"
done; done; done
