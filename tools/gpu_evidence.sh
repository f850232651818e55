# Round evidence run on a 4-GPU box: bench N=1/2/4, ncu of the N=1 kernel, size sweep, config 5, reference arm.
mkdir -p gpurun_out/ev
O=gpurun_out/ev
timeout 300 python bench.py > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log > $O/bench_n1.json
for N in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench$N rc $?"; tail -1 $O/bench_n$N.log > $O/bench_n$N.json
done
timeout 300 python bench.py --profile --steps 3 --warmup 2 --no-cpu > $O/prof_plain.log 2>&1; echo "prof plain rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file $O/launches.csv python bench.py --profile --steps 3 --warmup 2 --no-cpu > $O/ncu_list.log 2>&1; echo "ncu list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:r2_allreduce -s 3 -c 1 -o $O/sim8_full python bench.py --profile --steps 3 --warmup 2 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu full rc $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sizes.py > $O/sizes_n4.jsonl 2> $O/sizes_n4.err; echo "sizes rc $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/config5.py > $O/config5_n4.log 2>&1; echo "config5 rc $?"
timeout 300 python bench.py --impl reference > $O/ref_n1.log 2>&1; echo "ref rc $?"; tail -1 $O/ref_n1.log > $O/ref_n1.json
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"
