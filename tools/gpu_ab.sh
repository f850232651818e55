mkdir -p gpurun_out/ab
for p in SIMPLE LL; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$((RANDOM % 10)) tools/sweep_sizes.py --max-log2 26 --dtypes bf16 --protocol $p --no-nccl > gpurun_out/ab/$p.n4.jsonl 2> gpurun_out/ab/$p.n4.err; done
for p in SIMPLE LL; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$((RANDOM % 10)) tools/sweep_sizes.py --max-log2 26 --dtypes bf16 --protocol $p --no-nccl > gpurun_out/ab/$p.n2.jsonl 2> gpurun_out/ab/$p.n2.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29559 tools/sweep_sizes.py --max-log2 30 --dtypes bf16 > gpurun_out/ab/AUTO.n4.jsonl 2> gpurun_out/ab/AUTO.n4.err
echo done
