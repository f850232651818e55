# forced-protocol sweeps at N=2 and N=4 (alpha-beta refit) + AUTO sweep vs NCCL + tests
set -x
O=gpurun_out/ev11; mkdir -p $O
for N in 4 2; do
  for P in LL LL128 SIMPLE; do
    mx=28; [ $P = LL ] && mx=25; [ $P = LL128 ] && mx=27
    mn=10; [ $P = SIMPLE ] && mn=16
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --min-log2 $mn --max-log2 $mx --dtypes bf16 --protocol $P --no-nccl > $O/proto_${P}_n$N.jsonl 2>/dev/null
    python -c "
import json; print('N=$N $P', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in open('$O/proto_${P}_n$N.jsonl')])"
  done
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N tools/sweep_sizes.py --max-log2 28 --dtypes bf16 > $O/sizes_n$N.jsonl 2>/dev/null
  python -c "
import json
for l in open('$O/sizes_n$N.jsonl'):
    d = json.loads(l); print('N=$N', d['bytes'], d['protocol'], round(d['r2_ms']*1e3, 1), round(d['r2_busbw']), d.get('nccl_ms') and round(d['nccl_ms']*1e3, 1))"
done
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
