mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
python tools/sweep_grid.py 4 8:16:32768:512:16777216 8:16:8192:512:16777216 8:16:65536:512:67108864 8:16:16384:512:67108864 8:16:524288:512:268435456 8:16:131072:512:268435456 2>&1 | tee gpurun_out/sweep_chunk3.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sizes.py --max-log2 28 --dtypes bf16 > gpurun_out/sizes_n4.jsonl 2> gpurun_out/sizes_n4.err; echo "sizes rc $?"
