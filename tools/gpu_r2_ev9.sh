set -x
O=gpurun_out/ev9; mkdir -p $O
R=$PWD
for v in r1 new; do
  d=$R; [ $v != new ] && d=$R/ab/$v
  (cd $d && R2_TRACE=1 SIZES=1024,1024,1024,1024 PROTO=LL timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 tools/trace_multi.py > $R/$O/trace_$v.log 2>&1); grep "rank 0\]" $R/$O/trace_$v.log
done
for th in 256 512; do
R2_LL_THREADS=$th timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep_sizes.py --min-log2 20 --max-log2 26 --dtypes bf16 --protocol LL128 --no-nccl > $O/ll128_t$th.jsonl 2>/dev/null; echo "sizes rc $?"
python -c "
import json; print('$th', [(json.loads(l)['bytes']>>20, round(json.loads(l)['r2_ms']*1e3,1)) for l in open('$O/ll128_t$th.jsonl')])"
done
R2_LL_THREADS=512 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep_sizes.py --max-log2 20 --dtypes bf16 --protocol LL --no-nccl > $O/ll_t512.jsonl 2>/dev/null
python -c "
import json; print('LL512', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in open('$O/ll_t512.jsonl')])"
