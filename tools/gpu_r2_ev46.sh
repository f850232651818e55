# A/B: control-lane slot ring depth NSLOT 4 vs 8 (small/mid sizes and 256 MiB, N=4 and N=2)
O=gpurun_out/ev46; mkdir -p $O
for NS in 4 8 16; do
sed -i "s/^#define R2_NSLOT .*/#define R2_NSLOT $NS/" paper_2512_25059_b200/csrc/r2_kernels.cu
python -c "from paper_2512_25059_b200 import build as B; B.build()" || exit 1
echo "== NSLOT $NS"
for P in LL SIMPLE; do R2_TRACE=3 PROTO=$P SIM=4 timeout 120 python tools/trace_sim.py 2>&1 | tail -2; done
for N in 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --max-log2 28 --dtypes bf16 --no-nccl > $O/sizes_ns${NS}_n$N.jsonl 2>/dev/null; echo "sizes$N rc $?"
python -c "
import json
for l in open('$O/sizes_ns${NS}_n$N.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print('N=$N NS=$NS', d.get('bytes'), d.get('protocol'), round(d['r2_ms']*1e3,1))
" | paste - - - - | head -12
done
done
