mkdir -p gpurun_out
for s in BALANCE; do R2_DEBUG=1 STRATEGY=$s timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 tools/debug_multi.py > gpurun_out/dbg4_${s}.log 2>&1; echo "dbg rc $?"; grep "faulted call\|timeline\|published\|detect seq\|verdict round" gpurun_out/dbg4_${s}.log; done
M=268435456
python tools/sweep_grid.py 4 8:16:524288:512:$M 8:16:262144:512:$M 8:16:131072:512:$M 8:8:262144:512:$M 16:8:262144:512:$M 16:8:131072:512:$M 8:16:524288:256:$M 8:16:262144:1024:$M 8:16:524288:512:1073741824 8:16:262144:512:1073741824 2>&1 | tee gpurun_out/sweep4.log
