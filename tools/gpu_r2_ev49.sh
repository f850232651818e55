# NSLOT 8 vs 4 at 32 CTAs per GPU (K=8 x W=4, 512 KiB chunks) and at the headline, N=4 / N=2, same box
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for NS in 8 4 8 4; do
sed -i "s/^#define R2_NSLOT .*/#define R2_NSLOT $NS/" paper_2512_25059_b200/csrc/r2_kernels.cu
python -c "from paper_2512_25059_b200 import build as B; B.build()" || exit 1
for N in 4 2; do for W in 4 16; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --ctas $W --chunk 524288 $FL 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('NSLOT $NS N=$N W=$W', round(d['ms_per_step'],4), round(d['busbw_per_rank'],1))"
done; done; done
