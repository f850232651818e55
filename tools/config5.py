"""BASELINE configs[4]: Llama-3-8B-shaped gradient buckets, 640 x 25,000,000 B bf16,
with periodic fault injection (SURVEY reading C-18): a LINK fault on bucket
b = 0 (mod 64) (10 faults; rank, channel, step, chunk, offset drawn from a seeded
generator), REPAIR 32 buckets later.  Reports the total time of the 640 buckets
fault-free, faulted (Balance) and with NCCL; pass B re-runs the faulted schedule and
checks every bucket bit-identical to its fault-free result.

torchrun --nproc-per-node N tools/config5.py   |   python tools/config5.py (8 sim ranks)
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402

NB, BUCKET, POOL = 640, 25_000_000, 8


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    sim = world == 1
    n = 8 if sim else world
    count = BUCKET // 2
    W = 2 if sim else 16
    cfg = dict(nchannels=8, ctas_per_channel=W, max_bytes=BUCKET)
    if sim:
        comm = R.Comm(0, 1, 0, None, R.config_default(sim_ranks=n, **cfg))
        shape = (n, count)
        sync = torch.cuda.synchronize
        red = lambda x: x
    else:
        dist.init_process_group("gloo")
        comm = T.comm_from_env(R.config_default(**cfg))
        shape = (count,)

        def sync():
            torch.cuda.synchronize()
            dist.barrier()

        def red(x):
            t = torch.tensor([x], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
    g = torch.Generator(device="cuda")
    g.manual_seed(99 + rank)
    ins = [torch.randn(shape, generator=g, device="cuda").to(torch.bfloat16) for _ in range(POOL)]
    outs = [torch.empty_like(x) for x in ins]
    if not sim:
        for o in outs:
            T.register(comm, o)
    stream = torch.cuda.current_stream()

    def run_pass(check=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bad = torch.zeros((), dtype=torch.int64, device="cuda")
        e0.record(stream)
        for b in range(NB):
            T.allreduce(comm, ins[b % POOL], outs[b % POOL])
            if check is not None:
                bad += (outs[b % POOL] != check[b % POOL]).any()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1), int(bad.item())

    def arm_faults(base_seq):
        rng = np.random.default_rng(0xC5)
        K, m_guess = 8, 1
        for f in range(10):
            b = 64 * f
            comm.inject_fault(at_seq=base_seq + b, kind="LINK", src_rank=int(rng.integers(n)),
                              channel=int(rng.integers(K)), step=int(rng.integers(2 * n - 2)),
                              chunk=int(rng.integers(m_guess)), byte_offset=int(rng.integers(0, 64)) * 1024)
            for r in range(n):
                for c in range(K):
                    comm.inject_fault(at_seq=base_seq + b + 32, kind="REPAIR", src_rank=r, channel=c)

    for i in range(POOL):                       # warm-up + fault-free references
        T.allreduce(comm, ins[i], outs[i])
    sync()
    ref = [o.clone() for o in outs]
    sync()
    t_free, _ = run_pass()
    t_free = red(t_free)
    seq = comm.status()["seq"]
    arm_faults(seq + 1)
    sync()
    t_fault, _ = run_pass()
    t_fault = red(t_fault)
    rc = comm.sync()
    evs = comm.events()
    seq = comm.status()["seq"]
    arm_faults(seq + 1)
    sync()
    _, bad = run_pass(check=ref)
    bad = int(red(float(bad)))
    res = {"config": "640 x 25,000,000 B bf16 gradient buckets, 10 LINK faults (every 64), REPAIR +32",
           "ranks": n, "mode": "sim" if sim else "gpus", "total_ms_fault_free": t_free,
           "total_ms_faulted": t_fault, "per_fault_ms": (t_fault - t_free) / 10,
           "overhead_pct": 100 * (t_fault - t_free) / t_free, "rc": rc,
           "buckets_not_bit_identical": bad, "failover_ms_local": [e["failover_ms"] for e in evs],
           "roofline_total_ms_770": NB * 2 * (n - 1) / n * BUCKET / 770e9 * 1e3}
    if not sim:
        os.environ["NCCL_NVLS_ENABLE"] = "0"
        saved = os.dup(1)
        os.dup2(2, 1)
        pg = dist.new_group(backend="nccl")
        for i in range(POOL):
            dist.all_reduce(outs[i], group=pg)
        sync()
        os.dup2(saved, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for b in range(NB):
            dist.all_reduce(outs[b % POOL], group=pg)
        e1.record(stream)
        e1.synchronize()
        res["total_ms_nccl"] = red(e0.elapsed_time(e1))
        fo = [None] * world
        dist.all_gather_object(fo, res["failover_ms_local"])
        res["failover_ms"] = [x for part in fo for x in part]
    if rank == 0:
        print(json.dumps(res), flush=True)
    comm.finalize()


if __name__ == "__main__":
    main()
