set -x
O=gpurun_out/ev10; mkdir -p $O
timeout 300 python bench.py --no-cpu --no-e2e > $O/bench_n1.log 2>&1; echo "b1 rc $?"; tail -1 $O/bench_n1.log | cut -c1-330
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep_sizes.py --max-log2 28 --dtypes bf16 > $O/sizes_n4.jsonl 2>/dev/null; echo "sizes rc $?"
python - <<'PY'
import json
for l in open("gpurun_out/ev10/sizes_n4.jsonl"):
    d = json.loads(l); print(d["bytes"], d["protocol"], round(d["r2_ms"]*1e3, 1), round(d["r2_busbw"]), d.get("nccl_ms") and round(d["nccl_ms"]*1e3, 1))
PY
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -4 $O/pytest_gpu.log
