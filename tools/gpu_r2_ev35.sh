R=$PWD
for i in 1 2; do
for v in base tiny; do d=$R; [ $v != base ] && d=$R/ab/$v
(cd $d && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 tools/sweep_sizes.py --min-log2 20 --max-log2 25 --dtypes bf16 --protocol LL128 --no-nccl 2>/dev/null | python -c "
import json,sys; print('$v N=4', [(json.loads(l)['bytes']>>20, round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])")
done; done
for v in base tiny; do d=$R; [ $v != base ] && d=$R/ab/$v
(cd $d && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 tools/sweep_sizes.py --min-log2 20 --max-log2 25 --dtypes bf16 --protocol LL128 --no-nccl 2>/dev/null | python -c "
import json,sys; print('$v N=2', [(json.loads(l)['bytes']>>20, round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])")
done
