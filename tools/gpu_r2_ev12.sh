set -x
O=gpurun_out/ev12; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N tools/sweep_sizes.py --max-log2 30 --dtypes bf16,fp32 > $O/sizes_n$N.jsonl 2>/dev/null; echo "sizes $N rc $?"
  python -c "
import json
for l in open('$O/sizes_n$N.jsonl'):
    d = json.loads(l); print('N=$N', d['dtype'], d['bytes'], d['protocol'], round(d['r2_ms']*1e3, 1), round(d['r2_busbw']), d.get('nccl_ms') and round(d['nccl_ms']*1e3, 1))"
done
timeout 300 python tools/r2cc_stages.py > $O/r2cc_stages.log 2>&1; echo "stages rc $?"; cat $O/r2cc_stages.log | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:r2_ --csv --log-file $O/r2cc_launches.csv python tools/r2cc_stages.py > $O/r2cc_ncu.log 2>&1; echo "ncu rc $?"
