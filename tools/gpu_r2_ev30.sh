R=$PWD
for i in 1 2; do
for v in u4 u2; do d=$R; [ $v = u2 ] && d=$R/ab/u8
for N in 4 2; do
(cd $d && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --min-log2 22 --max-log2 27 --dtypes bf16 --protocol LL128 --no-nccl 2>/dev/null | python -c "
import json,sys; print('$v N=$N', [(json.loads(l)['bytes']>>20, round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])")
done; done; done
