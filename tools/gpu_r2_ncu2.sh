O=gpurun_out/ncu2; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:r2_ring -s 3 -c 1 -o $O/sim8_full python bench.py --profile --steps 3 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu full rc $?"
BCAST=0.529 timeout 300 python tools/r2cc_stages.py 2>&1 | tail -3
R2_R2CC_ONLY_STAGE=2 timeout 300 python tools/r2cc_stages.py 2>&1 | tail -1
