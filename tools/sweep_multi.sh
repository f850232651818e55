#!/bin/bash
# Tuning sweep of the multi-GPU path: CTAs per channel x chunk size.
# usage (on the GPU box): tools/sweep_multi.sh N "W list" "chunk list" [bytes]
N=${1:-2}; WS=${2:-"2 4 8"}; CHUNKS=${3:-"524288"}; BYTES=${4:-268435456}
for W in $WS; do for C in $CHUNKS; do
  out=$(timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 40 --warmup 5 --ctas $W --chunk $C \
        --bytes $BYTES --no-fault --no-e2e --no-nccl 2>/dev/null | tail -1)
  echo "$out" | python3 -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('N=$N W=$W chunk=$C ms=%.3f busbw=%.1f frac=%.3f' % (d['ms_per_step'], d['busbw_per_rank'], d['roofline']['frac']))
except Exception as e: print('N=$N W=$W chunk=$C failed', e)"
done; done
