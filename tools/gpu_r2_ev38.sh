O=gpurun_out/ev38; mkdir -p $O
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --max-log2 30 --dtypes bf16,fp32 > $O/sizes_n$N.jsonl 2>/dev/null; echo "sizes$N rc $?"
done
