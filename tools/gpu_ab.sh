# A/B of two builds of bench.py on the same box: ab/old (a git worktree of a
# previous commit, built) vs the working tree.  Usage: bash tools/gpu_ab.sh
set -x
O=gpurun_out/ab; mkdir -p $O
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for i in 1 2; do
  for v in old new; do
    d=.; [ $v = old ] && d=ab/old
    (cd $d && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$i bench.py --gpus 2 $FL) > $O/${v}_n2_$i.log 2>&1
    tail -1 $O/${v}_n2_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v n2 run $i', d['ms_per_step'], d['busbw_per_rank'])"
    (cd $d && timeout 300 python bench.py $FL) > $O/${v}_n1_$i.log 2>&1
    tail -1 $O/${v}_n1_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v n1 run $i', d['ms_per_step'])"
  done
done
