R2_TRACE=3 timeout 120 python tools/trace_sim.py 2>&1 | tail -1
R2_TRACE=3 PROTO=LL128 ELEMS=2097152 timeout 120 python tools/trace_sim.py 2>&1 | tail -1
python tools/sweep_sizes.py --sim-ranks 4 --ctas 4 --min-log2 10 --max-log2 11 --dtypes bf16 2>/dev/null | python -c "
import json,sys; print('period', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])"
