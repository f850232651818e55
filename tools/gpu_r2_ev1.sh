# Round-2 evidence on one GPU: GPU tests, smoke (plain and under ncu, as the
# driver runs it), bench N=1, launch list + full ncu capture of the bench
# kernel, compute-sanitizer memcheck of the simulated-rank path, reference arm.
set -x
O=gpurun_out/ev1; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -5 $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"; tail -2 $O/smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.log 2>&1; echo "smoke-ncu rc $?"; tail -3 $O/smoke_ncu.log
timeout 300 python bench.py > $O/bench_n1.log 2>&1; echo "bench1 rc $?"; tail -1 $O/bench_n1.log > $O/bench_n1.json; cut -c1-800 $O/bench_n1.json
timeout 300 python bench.py --profile --steps 3 --warmup 3 --no-cpu > $O/prof_plain.log 2>&1; echo "prof plain rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --profile --steps 3 --warmup 3 --no-cpu > $O/ncu_list.log 2>&1; echo "ncu list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:r2_allreduce -s 3 -c 1 -o $O/sim8_full python bench.py --profile --steps 3 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu full rc $?"
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_sim.py > $O/memcheck.log 2>&1; echo "memcheck rc $?"; tail -5 $O/memcheck.log
timeout 300 python bench.py --impl reference > $O/ref_n1.log 2>&1; echo "ref rc $?"; tail -1 $O/ref_n1.log > $O/ref_n1.json
