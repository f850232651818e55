# LL128 bring-up + multi-GPU regression hunt (4-GPU box)
set -x
O=gpurun_out/l128; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ll128_tear tools/ll128_tear.cu
timeout 60 tools/bin/ll128_tear 5 4096 > $O/tear.log 2>&1; echo "tear rc $?"; cat $O/tear.log
timeout 60 tools/bin/ll128_tear 5 64 >> $O/tear.log 2>&1; echo "tear2 rc $?"; tail -1 $O/tear.log
(nvidia-smi nvlink -h; nvidia-smi nvlink -gt d -i 0; nvidia-smi nvlink -s -i 0) > $O/nvsmi_nvlink.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ll.py -x -q > $O/pytest_ll.log 2>&1; echo "ll rc $?"; tail -15 $O/pytest_ll.log
FL="--profile --no-fault --no-e2e --no-cpu --no-nccl --no-coll --steps 100 --warmup 10"
for i in 1 2; do
  for v in r1 svc gen new; do
    d=.; [ $v != new ] && d=ab/$v
    (cd $d && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954$i bench.py --gpus 4 $FL) > $O/${v}_n4_$i.log 2>&1
    tail -1 $O/${v}_n4_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v n4 run $i', d['ms_per_step'], d['busbw_per_rank'])"
  done
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $O/pytest_multi.log 2>&1; echo "multi rc $?"; tail -5 $O/pytest_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sizes.py --max-log2 28 --dtypes bf16 > $O/sizes_n4.jsonl 2> $O/sizes_n4.err; echo "sizes rc $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep_sizes.py --max-log2 27 --dtypes bf16 --protocol LL128 --no-nccl > $O/sizes_n4_ll128.jsonl 2> $O/sizes_n4_ll128.err; echo "sizes128 rc $?"
python - <<'PY'
import json
for f in ("gpurun_out/l128/sizes_n4.jsonl", "gpurun_out/l128/sizes_n4_ll128.jsonl"):
    print(f)
    try:
        for l in open(f):
            d = json.loads(l); print(d["bytes"], d["protocol"], round(d["r2_ms"]*1e3, 1), round(d["r2_busbw"]), d.get("nccl_ms") and round(d["nccl_ms"]*1e3, 1))
    except Exception as e: print(e)
PY
