set -x
O=gpurun_out/fin3; mkdir -p $O
for N in 4 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench$N rc $?"; tail -1 $O/bench_n$N.log > $O/bench_n$N.json
python -c "
import json; d=json.load(open('$O/bench_n$N.json')); r=d['roofline']
print('N=$N', d['ms_per_step'], round(d['busbw_per_rank'],1), round(r['frac'],3), (d.get('nccl_same_box') or {}).get('busbw_per_gpu'))
print(json.dumps(d.get('bucket_25MB'))[:2500])"
done
timeout 400 python bench.py > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log > $O/bench_n1.json
