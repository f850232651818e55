set -x
O=gpurun_out/ev26; mkdir -p $O
for N in 4 2; do
for P in SIMPLE LL128; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --min-log2 22 --max-log2 28 --dtypes bf16 --protocol $P --no-nccl > $O/${P}_n$N.jsonl 2>/dev/null
python -c "
import json; print('$P N=$N', [(json.loads(l)['bytes']>>20, round(json.loads(l)['r2_ms']*1e3,1)) for l in open('$O/${P}_n$N.jsonl')])"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --no-e2e --no-coll --no-fault --no-cpu > $O/bench_n$N.log 2>&1
python -c "
import json; d=json.loads(open('$O/bench_n$N.log').read().strip().split(chr(10))[-1]); print('bench N=$N', d['ms_per_step'], round(d['busbw_per_rank'],1), (d.get('nccl_same_box') or {}).get('busbw_per_gpu'))"
done
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
