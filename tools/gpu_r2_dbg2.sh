# LL128 fault debug (1 GPU) + perf regression A/B at N=4
set -x
O=gpurun_out/dbg2; mkdir -p $O
timeout 600 python tools/debug_ll128.py > $O/debug_ll128.log 2>&1; echo "dbg rc $?"; head -60 $O/debug_ll128.log
PROTO=LL timeout 300 python tools/debug_ll128.py > $O/debug_ll.log 2>&1; echo "dbg-ll rc $?"; grep -c "bad_ranks={}" $O/debug_ll.log
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for i in 1 2; do
  for v in gen d48 newnonvml new; do
    d=.; E=""; [ $v = gen ] && d=ab/gen; [ $v = d48 ] && d=ab/d48; [ $v = newnonvml ] && E="R2_BENCH_NO_NVML=1"
    (cd $d && env $E timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954$i bench.py --gpus 4 $FL) > $O/${v}_n4_$i.log 2>&1
    tail -1 $O/${v}_n4_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v n4 run $i', d['ms_per_step'], d['busbw_per_rank'])"
  done
done
