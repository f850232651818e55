# Round-2 evidence (4-GPU box): tests, smoke (plain + ncu), bench N=1/2/4, ncu of the N=1 kernel,
# size sweeps N=2/4, config 5 at N=4, reference arm
set -x
O=gpurun_out/fin9; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $O/smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.log 2>&1; echo "smoke-ncu rc $?"; tail -1 $O/smoke_ncu.log
timeout 400 python bench.py > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log > $O/bench_n1.json
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench$N rc $?"; tail -1 $O/bench_n$N.log > $O/bench_n$N.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --profile --steps 3 --warmup 3 --no-cpu > $O/ncu_list.log 2>&1; echo "ncu list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:r2_ring -s 3 -c 1 -o $O/sim8_full python bench.py --profile --steps 3 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu full rc $?"
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --max-log2 30 --dtypes bf16,fp32 > $O/sizes_n$N.jsonl 2>/dev/null; echo "sizes$N rc $?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/config5.py > $O/config5_n4.log 2>&1; echo "config5 rc $?"; tail -2 $O/config5_n4.log
timeout 300 python bench.py --impl reference > $O/ref_n1.log 2>&1; echo "ref rc $?"; tail -1 $O/ref_n1.log > $O/ref_n1.json
python - <<'PY'
import json
for n in (1, 2, 4):
    try:
        d = json.load(open(f"gpurun_out/fin9/bench_n{n}.json")); r = d["roofline"]
        print(n, d["ms_per_step"], round(d["value"], 1), round(r["frac"], 3), r.get("traffic_over_algorithmic"), (d.get("e2e") or {}).get("value"),
              (d.get("small_footprint") or {}).get("busbw_per_rank"), (d.get("nccl_same_box") or {}).get("busbw_per_gpu"))
    except Exception as e: print(n, e)
PY
