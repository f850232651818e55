# full GPU suite (1/2/4 GPUs) + small-size floor A/B (r1 vs now) + host enqueue cost + trace
set -x
O=gpurun_out/ev6; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -15 $O/pytest_gpu.log
for v in r1 new; do
  d=.; [ $v = r1 ] && d=ab/r1
  (cd $d && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sizes.py --max-log2 22 --dtypes bf16 --no-nccl > ../../$O/floor_${v}.jsonl 2>/dev/null || true)
  [ $v = new ] && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sizes.py --max-log2 22 --dtypes bf16 --no-nccl > $O/floor_new.jsonl 2>/dev/null
done
python - <<'PY'
import json
for v in ("r1", "new"):
    try:
        print(v, [(json.loads(l)["bytes"], json.loads(l)["protocol"], round(json.loads(l)["r2_ms"] * 1e3, 1)) for l in open(f"gpurun_out/ev6/floor_{v}.jsonl")])
    except Exception as e: print(v, e)
PY
R2_DEBUG=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/host_overhead.py > $O/host_overhead.log 2>&1; echo "host rc $?"; grep -i "enqueue\|per call\|us" $O/host_overhead.log | head -12
R2_TRACE=2 SIZES=1024 PROTO=LL timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 tools/trace_multi.py > $O/trace_ll.log 2>&1; echo "trace rc $?"; grep "rank" $O/trace_ll.log | head -8
