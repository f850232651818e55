python tools/sweep_sizes.py --sim-ranks 4 --ctas 4 --min-log2 10 --max-log2 11 --dtypes bf16 2>/dev/null | python -c "
import json,sys; print('sim period', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep_sizes.py --max-log2 16 --dtypes bf16 --no-nccl 2>/dev/null | python -c "
import json,sys; print('N=4', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
