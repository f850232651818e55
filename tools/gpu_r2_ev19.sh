set -x
O=gpurun_out/ev19; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --min-log2 20 --max-log2 30 --dtypes bf16 > $O/sizes_n$N.jsonl 2>/dev/null; echo "sizes$N rc $?"
python -c "
import json
for l in open('$O/sizes_n$N.jsonl'):
    d = json.loads(l); print('N=$N', d['bytes']>>20, d['protocol'], round(d['r2_ms']*1e3, 1), round(d['r2_busbw']), d.get('nccl_ms') and round(d['nccl_ms']*1e3, 1))"
done
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --min-log2 22 --max-log2 28 --dtypes bf16 --protocol SIMPLE --no-nccl > $O/simple_n$N.jsonl 2>/dev/null
python -c "
import json; print('SIMPLE N=$N', [(json.loads(l)['bytes']>>20, round(json.loads(l)['r2_ms']*1e3,1)) for l in open('$O/simple_n$N.jsonl')])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --min-log2 20 --max-log2 27 --dtypes bf16 --protocol LL128 --no-nccl > $O/ll128_n$N.jsonl 2>/dev/null
python -c "
import json; print('LL128 N=$N', [(json.loads(l)['bytes']>>20, round(json.loads(l)['r2_ms']*1e3,1)) for l in open('$O/ll128_n$N.jsonl')])"
done
BCAST=0.529 timeout 300 python tools/r2cc_stages.py 2>&1 | tail -3
