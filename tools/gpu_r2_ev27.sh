run() { python tools/sweep_sizes.py --sim-ranks 4 --ctas 4 --min-log2 10 --max-log2 11 --dtypes bf16 2>/dev/null | python -c "
import json,sys; print('$1', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])"; }
run coop; R2_PLAIN_LAUNCH=1 run plain; R2_NO_SERVICE_CTA=1 R2_PLAIN_LAUNCH=1 run plain-nosvc
for v in coop plain; do E=""; [ $v = plain ] && E="R2_PLAIN_LAUNCH=1"
env $E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep_sizes.py --max-log2 24 --dtypes bf16 --no-nccl 2>/dev/null | python -c "
import json,sys; print('$v N=4', [(json.loads(l)['bytes']>>10, json.loads(l)['protocol'], round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])"
done
