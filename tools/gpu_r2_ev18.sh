O=gpurun_out/ev18; mkdir -p $O
timeout 120 python tools/trace_sim.py 2>&1 | tail -2
python tools/sweep_sizes.py --sim-ranks 4 --ctas 4 --min-log2 10 --max-log2 11 --dtypes bf16 2>/dev/null | python -c "
import json,sys; print('period', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:r2_ring -s 40 -c 1 -o $O/ll_small python tools/sweep_sizes.py --sim-ranks 8 --ctas 2 --min-log2 12 --max-log2 12 --dtypes bf16 > $O/ncu.log 2>&1; echo "ncu rc $?"
