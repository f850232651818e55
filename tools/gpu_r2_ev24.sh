set -x
O=gpurun_out/ev24; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ll.py tests/test_gpu_rerank.py -q -x > $O/pytest_ll.log 2>&1; echo "ll rc $?"; tail -5 $O/pytest_ll.log
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -4 $O/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --no-e2e --no-coll > $O/bench_n4.log 2>&1; echo "bench4 rc $?"
python -c "
import json; d=json.loads(open('$O/bench_n4.log').read().strip().split(chr(10))[-1]); print(d['ms_per_step'], d['busbw_per_rank']); b=d.get('bucket_25MB') or {}
print(b.get('ms'), b.get('nccl_ms'), (b.get('fault_unpaced') or {}).get('degraded_over_bound'), (b.get('fault_paced') or {}).get('degraded_over_bound'), (b.get('fault_unpaced') or {}).get('bit_identical_to_healthy'))"
