"""BASELINE configs[1]: allreduce sweep 1 KiB - 1 GiB, fp32/bf16, r2 vs NCCL.

torchrun --nproc-per-node N tools/sweep_sizes.py [--max-log2 30] [--dtypes bf16,fp32]
or plain `python tools/sweep_sizes.py` for the 1-GPU simulated-rank mode (8 ranks).
Rank 0 prints one JSON line per (dtype, size); busbw per rank (nccl-tests).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402


def timed(fn, iters, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--dtypes", default="bf16,fp32")
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--sim-ranks", type=int, default=8)
    ap.add_argument("--protocol", default="AUTO", choices=["AUTO", "SIMPLE", "LL", "LL128"])
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--ll-max", type=int, default=128 << 20, help="ll_max_bytes (line-protocol scratch)")
    ap.add_argument("--threads", type=int, default=0, help="threads per CTA (0 = 512 sim / 256 GPUs, as bench.py)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    maxb = 1 << a.max_log2
    sim = world == 1
    n = a.sim_ranks if sim else world
    W = a.ctas or (2 if sim else 16)
    if sim:
        comm = R.Comm(0, 1, 0, None, R.config_default(sim_ranks=n, nchannels=8, ctas_per_channel=W, protocol=a.protocol,
                                                      max_bytes=maxb))
        reduce_max = lambda x: x
        barrier = torch.cuda.synchronize
    else:
        dist.init_process_group("gloo")
        comm = T.comm_from_env(R.config_default(nchannels=8, ctas_per_channel=W, max_bytes=maxb, protocol=a.protocol,
                                                ll_max_bytes=min(maxb, a.ll_max), threads_per_cta=a.threads or 256))
        os.environ["NCCL_NVLS_ENABLE"] = "0"
        saved = os.dup(1)
        os.dup2(2, 1)
        pg = dist.new_group(backend="nccl")
        dist.all_reduce(torch.ones(1, device="cuda"), group=pg)
        torch.cuda.synchronize()
        os.dup2(saved, 1)

        def reduce_max(x):
            t = torch.tensor([x], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        def barrier():
            torch.cuda.synchronize()
            dist.barrier()
    stream = torch.cuda.current_stream()
    for dt in a.dtypes.split(","):
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        E = 2 if dt == "bf16" else 4
        rows = n if sim else 1
        send = torch.randn((rows, maxb // E), device="cuda").to(tdt)
        recv = torch.empty_like(send)
        if not sim:
            T.register(comm, recv)
        for lg in range(a.min_log2, a.max_log2 + 1):
            S = 1 << lg
            cnt = S // E
            if sim:
                s2 = send[:, :cnt].contiguous()
                r2 = torch.empty_like(s2)
                fn = lambda: T.allreduce(comm, s2, r2)
            else:
                fn = lambda: comm.allreduce(send.data_ptr(), recv.data_ptr(), cnt, R.BFLOAT16 if dt == "bf16"
                                            else R.FLOAT32, stream.cuda_stream)
            iters = max(5, min(200, (1 << 27) // S))
            for _ in range(3):
                fn()
            barrier()
            ms = reduce_max(timed(fn, iters, stream))
            assert comm.sync() == R.SUCCESS
            out = {"dtype": dt, "bytes": S, "ranks": n, "mode": "sim" if sim else "gpus", "r2_ms": ms,
                   "r2_busbw": 2 * (n - 1) / n * S / (ms * 1e-3) / 1e9, "protocol": comm.status()["last_protocol"]}
            if not sim and not a.no_nccl:
                buf = send[0, :cnt] if send.dim() == 2 else send[:cnt]
                f2 = lambda: dist.all_reduce(buf, group=pg)
                for _ in range(3):
                    f2()
                barrier()
                msn = reduce_max(timed(f2, iters, stream))
                out.update(nccl_ms=msn, nccl_busbw=2 * (n - 1) / n * S / (msn * 1e-3) / 1e9)
            if rank == 0:
                print(json.dumps(out), flush=True)
            barrier()
    comm.finalize()
    if not sim:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
