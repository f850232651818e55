timeout 120 python tools/trace_sim.py 2>&1 | tail -2
python tools/sweep_sizes.py --sim-ranks 4 --ctas 4 --min-log2 10 --max-log2 11 --dtypes bf16 2>/dev/null | python -c "
import json,sys; print('period', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])"
timeout 900 python -m pytest tests/test_gpu_ll.py tests/test_gpu_sim.py tests/test_gpu_rsag.py -q -x 2>&1 | tail -2
