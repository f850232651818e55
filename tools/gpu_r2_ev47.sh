# A/B: 16-byte aligned Slot / Meta (NSLOT 8)
O=gpurun_out/ev47; mkdir -p $O
for AL in "__align__(16)" " "; do
sed -i "s/^#define R2_SLOT_ALIGN .*/#define R2_SLOT_ALIGN $AL/" paper_2512_25059_b200/csrc/r2_kernels.cu
python -c "from paper_2512_25059_b200 import build as B; B.build()" || exit 1
echo "== ALIGN '$AL'"
for P in LL SIMPLE; do R2_TRACE=3 PROTO=$P SIM=4 timeout 120 python tools/trace_sim.py 2>&1 | tail -2; done
for N in 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/sweep_sizes.py --max-log2 26 --dtypes bf16 --no-nccl 2>/dev/null | python -c "
import json,sys
print(' '.join(str(round(json.loads(l)['r2_ms']*1e3,1)) for l in sys.stdin if l.startswith('{')))"
done
done
