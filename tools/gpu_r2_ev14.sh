O=gpurun_out/ev14; mkdir -p $O
R=$PWD
run() { python tools/sweep_sizes.py --sim-ranks 4 --ctas ${2:-4} --min-log2 10 --max-log2 11 --dtypes bf16 2>/dev/null | python -c "
import json,sys; print('$1', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin])"; }
for i in 1 2; do
(cd ab/r1 && run r1)
run new
R2_NO_SERVICE_CTA=1 run new-nosvc
run new-W1 1
R2_NO_SERVICE_CTA=1 run new-nosvc-W1 1
(cd ab/r1 && run r1-W1 1)
done
