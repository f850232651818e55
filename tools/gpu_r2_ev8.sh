set -x
O=gpurun_out/ev8; mkdir -p $O
R=$PWD
for v in r1 new; do
  d=$R; [ $v != new ] && d=$R/ab/$v
  (cd $d && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sizes.py --max-log2 14 --dtypes bf16 --no-nccl > $R/$O/floor_${v}.jsonl 2>/dev/null)
  python -c "
import json; print('$v', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in open('$R/$O/floor_${v}.jsonl')])"
done
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -4 $O/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep_sizes.py --max-log2 28 --dtypes bf16 > $O/sizes_n4.jsonl 2>/dev/null; echo "sizes rc $?"
python - <<'PY'
import json
for l in open("gpurun_out/ev8/sizes_n4.jsonl"):
    d = json.loads(l); print(d["bytes"], d["protocol"], round(d["r2_ms"]*1e3, 1), round(d["r2_busbw"]), d.get("nccl_ms") and round(d["nccl_ms"]*1e3, 1))
PY
timeout 300 python bench.py --profile --protocol LL128 --bytes 16777216 --steps 3 --warmup 3 --no-cpu > $O/prof_ll128.log 2>&1; echo "prof rc $?"; tail -1 $O/prof_ll128.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:r2_allreduce -s 3 -c 1 -o $O/ll128_sim python bench.py --profile --protocol LL128 --bytes 16777216 --steps 3 --warmup 3 --no-cpu > $O/ncu_ll128.log 2>&1; echo "ncu rc $?"
