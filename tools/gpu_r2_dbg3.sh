set -x
O=gpurun_out/dbg3; mkdir -p $O
timeout 600 python tools/debug_ll128.py > $O/debug_ll128.log 2>&1; echo "dbg rc $?"; grep -c "bad_ranks={}" $O/debug_ll128.log; grep -v "bad_ranks={}" $O/debug_ll128.log | head -20
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/debug_multi2.py > $O/multi2.log 2>&1; echo "multi2 rc $?"; grep "rerank=" $O/multi2.log; tail -5 $O/multi2.log
timeout 900 python -m pytest tests/test_gpu_rerank.py tests/test_gpu_ll.py -x -q > $O/pytest.log 2>&1; echo "pytest rc $?"; tail -5 $O/pytest.log
