# SIMPLE input word: relaxed polls + one acquire (0) vs acquire polls (1), alternating on one box
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for AQ in 0 1 0 1; do
sed -i "s/^#define R2_ACQ_POLL .*/#define R2_ACQ_POLL $AQ/" paper_2512_25059_b200/csrc/r2_kernels.cu
python -c "from paper_2512_25059_b200 import build as B; B.build()" || exit 1
for N in 2 4; do for S in 268435456 67108864; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --bytes $S --protocol SIMPLE $FL 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ACQ_POLL $AQ N=$N S=$S', round(d['ms_per_step'],4), round(d['busbw_per_rank'],1))"
done; done; done
