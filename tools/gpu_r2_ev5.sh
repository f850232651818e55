# LL128 fix check + full GPU suite (incl. 2/4-GPU parity) + N=4 size sweep + bench N=4
set -x
O=gpurun_out/ev5; mkdir -p $O
timeout 600 python tools/debug_ll128.py > $O/debug_ll128.log 2>&1; echo "dbg rc $?"; grep -c "bad_ranks={}" $O/debug_ll128.log; grep -v "bad_ranks={}" $O/debug_ll128.log | head -20
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -15 $O/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sizes.py --max-log2 28 --dtypes bf16 > $O/sizes_n4.jsonl 2> $O/sizes_n4.err; echo "sizes rc $?"
python - <<'PY'
import json
for l in open("gpurun_out/ev5/sizes_n4.jsonl"):
    d = json.loads(l); print(d["bytes"], d["protocol"], round(d["r2_ms"]*1e3, 1), round(d["r2_busbw"]), d.get("nccl_ms") and round(d["nccl_ms"]*1e3, 1))
PY
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --per-step > $O/bench_n4.log 2>&1; echo "bench4 rc $?"; tail -1 $O/bench_n4.log > $O/bench_n4.json; grep "per-step" $O/bench_n4.log
python -c "
import json; d=json.load(open('gpurun_out/ev5/bench_n4.json')); r=d['roofline']
print(d['ms_per_step'], d['busbw_per_rank'], r['frac'], r.get('traffic_over_algorithmic'), d.get('small_footprint'), d.get('nccl_same_box',{}).get('busbw_per_gpu'))
print(json.dumps(d.get('rerank'))); print(json.dumps(d.get('r2cc_allreduce'))[:800])"
