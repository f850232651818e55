mkdir -p gpurun_out/fin
O=gpurun_out/fin
timeout 300 python bench.py > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log > $O/bench_n1.json
for N in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench$N rc $?"; tail -1 $O/bench_n$N.log > $O/bench_n$N.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/config5.py > $O/config5_n4.log 2>&1; echo "config5 rc $?"
timeout 300 python bench.py --impl reference > $O/ref_n1.log 2>&1; echo "ref rc $?"; tail -1 $O/ref_n1.log
