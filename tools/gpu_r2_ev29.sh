set -x
O=gpurun_out/ev29; mkdir -p $O
R2_TRACE=3 timeout 120 python tools/trace_sim.py 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep_sizes.py --max-log2 26 --dtypes bf16 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['bytes'], d['protocol'], round(d['r2_ms']*1e3,1), round(d['nccl_ms']*1e3,1))"
