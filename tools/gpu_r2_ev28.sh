set -x
O=gpurun_out/ev28; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_r2cc.py tests/test_oracle_r2cc.py -q > $O/pytest.log 2>&1; echo "rc $?"; tail -2 $O/pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --no-e2e --no-coll > $O/bench_n4.log 2>&1; echo "bench4 rc $?"
python -c "
import json; d=json.loads(open('$O/bench_n4.log').read().strip().split(chr(10))[-1]); print(json.dumps(d.get('r2cc_allreduce')))"
