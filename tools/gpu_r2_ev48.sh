O=gpurun_out/ev48; mkdir -p $O
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench$N rc $?"; tail -1 $O/bench_n$N.log > $O/bench_n$N.json
done
python - <<'PY'
import json
for n in (2, 4):
    d = json.load(open(f"gpurun_out/ev48/bench_n{n}.json")); r = d["roofline"]
    print(n, d["ms_per_step"], round(d["value"], 1), round(r["frac"], 3), (d.get("small_footprint") or {}).get("busbw_per_rank"), (d.get("nccl_same_box") or {}).get("busbw_per_gpu"), d["bucket_25MB"]["ms"], d["bucket_25MB"].get("nccl_ms"))
PY
