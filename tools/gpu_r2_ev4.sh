# Round-2 multi-GPU evidence (4-GPU box): NVML NVLink counter check, the
# multi-GPU parity tests (world 2 and 4), bench N=2 and N=4 (NVLink counters,
# 32-CTA line).
set -x
O=gpurun_out/ev4; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 120 python tools/nvlink_probe.py > $O/nvlink_probe.log 2>&1; echo "probe rc $?"; tail -14 $O/nvlink_probe.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -rs > $O/pytest_multi.log 2>&1; echo "multi rc $?"; tail -4 $O/pytest_multi.log
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench$N rc $?"; tail -1 $O/bench_n$N.log > $O/bench_n$N.json
python -c "
import json; d=json.load(open('$O/bench_n$N.json')); r=d['roofline']
print('N=$N', d['ms_per_step'], round(d['busbw_per_rank'],1), 'frac', round(r['frac'],3), 'traffic', r.get('traffic'), r.get('traffic_over_algorithmic'))
print(json.dumps(r.get('nvlink_counters_per_rank'))[:1500]); print(json.dumps(d.get('small_footprint')))"
done
