set -x
O=gpurun_out/ev32; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --max-log2 28 --dtypes bf16 > $O/sizes_n$N.jsonl 2>/dev/null
python -c "
import json
for l in open('$O/sizes_n$N.jsonl'):
    d=json.loads(l); print('N=$N', d['bytes'], d['protocol'], round(d['r2_ms']*1e3,1), round(d['nccl_ms']*1e3,1))"
done
