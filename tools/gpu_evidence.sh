# Round evidence run on a 4-GPU box: bench N=1/2/4, ncu of the N=1 kernel, size sweep, P2P peak.
mkdir -p gpurun_out/ev
O=gpurun_out/ev
timeout 300 python bench.py > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log > $O/bench_n1.json
for N in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench$N rc $?"; tail -1 $O/bench_n$N.log > $O/bench_n$N.json
done
timeout 300 python bench.py --profile --steps 3 --warmup 2 --no-cpu > $O/prof_plain.log 2>&1; echo "prof plain rc $?"
if [ -s $O/prof_plain.log ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file $O/launches.csv python bench.py --profile --steps 3 --warmup 2 --no-cpu > $O/ncu_list.log 2>&1; echo "ncu list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:r2_allreduce -s 3 -c 1 -o $O/sim8_full python bench.py --profile --steps 3 --warmup 2 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu full rc $?"
fi
./tools/bin/p2p_bw 4 256 > $O/p2p4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sizes.py > $O/sizes_n4.jsonl 2> $O/sizes_n4.err; echo "sizes rc $?"
