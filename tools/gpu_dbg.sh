mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
for s in BALANCE HOT_REPAIR; do for i in 1; do R2_DEBUG=1 STRATEGY=$s timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 tools/debug_multi.py > gpurun_out/dbg4_${s}_$i.log 2>&1; echo "dbg rc $?"; grep "faulted call\|timeline\|published\|detect seq" gpurun_out/dbg4_${s}_$i.log; done; done
