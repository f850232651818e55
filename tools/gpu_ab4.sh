# A/B/C of builds at N=4 (ab/r1 = round-1 final, ab/old = service CTA commit, . = working tree)
set -x
O=gpurun_out/ab4; mkdir -p $O
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for i in 1 2; do
  for v in r1 old new; do
    d=.; [ $v = old ] && d=ab/old; [ $v = r1 ] && d=ab/r1
    (cd $d && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954$i bench.py --gpus 4 $FL) > $O/${v}_n4_$i.log 2>&1
    tail -1 $O/${v}_n4_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v n4 run $i', d['ms_per_step'], d['busbw_per_rank'])"
  done
done
python tools/nvlink_probe.py > $O/nvlink_probe.log 2>&1; cat $O/nvlink_probe.log
